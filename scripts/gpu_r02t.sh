#!/bin/bash
# round 2 pass t: lean + packed FP32x2 tiles -- the -m gpu suite; A/B of the default build
# (lean, packed, unroll 2) against pk16 (packed, full unroll), nopack (lean scalar) and
# nolean (round-2 folded slots); SASS source profiles of 3ce3 (lean vs nolean) and 7cpa
set -u
OUT=gpurun_out/r02t; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
bash scripts/gpu_ab.sh $OUT/ab "7cpa 3ce3" "pk16 nopack nolean" 2
prof() {   # prof <tag> <config> <lib>
  DOCK_LIB=$3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ls_adadelta -s 3 -c 1 \
      -o /tmp/p_$1 python bench.py --config $2 --steps 1 --warmup 0 --no-cpu --no-parts > $OUT/ncu_$1.log 2>&1
  python scripts/ncu_summary.py full /tmp/p_$1.ncu-rep > $OUT/full_$1.txt 2>&1
  ncu -i /tmp/p_$1.ncu-rep --page source --csv --print-source sass > $OUT/sass_$1.csv 2>&1
  gzip -f $OUT/sass_$1.csv
  python scripts/sass_blocks.py $OUT/sass_$1.csv.gz 30 > $OUT/blocks_$1.txt 2>&1
  head -12 $OUT/full_$1.txt; head -8 $OUT/blocks_$1.txt
}
prof 3ce3_lean 3ce3 ""
prof 3ce3_nolean 3ce3 build/ab/libdock_nolean.so
prof 7cpa_packed 7cpa ""
