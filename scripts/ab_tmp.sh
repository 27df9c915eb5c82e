#!/bin/bash
set -u
OUT=gpurun_out/ab10; mkdir -p $OUT
bash scripts/gpu_tests.sh ab10t
cap() {  # tag kernel-regex skip cmd...
  local tag=$1 re=$2 skip=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o /tmp/$tag "$@" > $OUT/ncu_$tag.log 2>&1
  python scripts/ncu_summary.py full /tmp/$tag.ncu-rep > $OUT/full_$tag.txt 2>&1
  ncu -i /tmp/$tag.ncu-rep --page source --csv --print-source sass > $OUT/sass_$tag.csv 2>/dev/null; gzip -f $OUT/sass_$tag.csv
  rm -f /tmp/$tag.ncu-rep
  echo "captured $tag: $(grep -m1 kernel $OUT/full_$tag.txt)"
}
cap ls_7cpa k_ls_adadelta 5 python bench.py --config 7cpa --steps 1 --warmup 0 --no-cpu
