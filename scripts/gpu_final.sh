#!/bin/bash
# Full evidence pass: tests, smoke, bench lines (+ CPU baselines), ncu launch lists and
# full captures of the LS kernels, microbenchmarks with summarised ncu captures.
set -u
TAG=${1:-final}
bash scripts/gpu_round.sh $TAG 1stp 3ce3 7cpa hts
OUT=gpurun_out/$TAG
for C in 1stp 3ce3 7cpa; do
  timeout 300 python bench.py --micro --config $C --steps 3 > $OUT/micro_$C.json 2>$OUT/micro_$C.err; tail -c 300 $OUT/micro_$C.json
done
cap() {  # tag kernel-regex skip cmd...
  local tag=$1 re=$2 skip=$3; shift 3
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o /tmp/$tag "$@" > $OUT/ncu_$tag.log 2>&1
  python scripts/ncu_summary.py full /tmp/$tag.ncu-rep > $OUT/full_$tag.txt 2>&1
  rm -f /tmp/$tag.ncu-rep
  echo "captured $tag: $(grep -m1 kernel $OUT/full_$tag.txt)"
}
cap micro_inter_7cpa k_bench_part 0 python bench.py --micro --config 7cpa --steps 1 --micro-iters 5
cap micro_intra_7cpa k_bench_part 3 python bench.py --micro --config 7cpa --steps 1 --micro-iters 5
cap micro_inter_1stp k_bench_part 0 python bench.py --micro --config 1stp --steps 1 --micro-iters 5
cap micro_intra_1stp k_bench_part 3 python bench.py --micro --config 1stp --steps 1 --micro-iters 5
cap ls_3ce3 k_ls_adadelta 5 python bench.py --config 3ce3 --steps 1 --warmup 0 --no-cpu
du -sh gpurun_out
