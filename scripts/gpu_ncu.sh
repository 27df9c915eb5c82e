#!/bin/bash
# ncu captures summarised on the box (raw counters + SASS source view as CSV); the
# .ncu-rep files are deleted to stay under gpurun's 64 MiB copy-back limit.
set -u
OUT=gpurun_out/${1:-ncu}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
cap() {  # tag kernel-regex skip cmd...
  local tag=$1 re=$2 skip=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o /tmp/$tag "$@" > $OUT/ncu_$tag.log 2>&1
  python scripts/ncu_summary.py full /tmp/$tag.ncu-rep > $OUT/full_$tag.txt 2>&1
  ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > $OUT/sass_$tag.csv 2>/dev/null
  gzip -f $OUT/sass_$tag.csv
  echo "captured $tag: $(grep -m1 kernel $OUT/full_$tag.txt)"
}
cap 7cpa_ada k_ls_adadelta 5 python bench.py --config 7cpa --steps 1 --warmup 0 --no-cpu
cap 3ce3_ada k_ls_adadelta 5 python bench.py --config 3ce3 --steps 1 --warmup 0 --no-cpu
cap 7cpa_intra k_bench_part 3 python bench.py --micro --config 7cpa --steps 1 --micro-iters 5
cap 7cpa_inter k_bench_part 0 python bench.py --micro --config 7cpa --steps 1 --micro-iters 5
cap 1stp_tree k_ls_sw 20 python bench.py --config 1stp --steps 1 --warmup 0 --no-cpu
ls -la $OUT
