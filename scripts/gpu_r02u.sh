#!/bin/bash
# round 2 pass u: packed FP32x2 tiles as a compile-time kernel variant (PK) with the lean
# constants only in the packed rows, the H-bond side list summed per atom by a segmented
# scan -- the -m gpu suite, A/B against DK_PACKED=0 (nopk), SASS profile of 7cpa
set -u
OUT=gpurun_out/r02u; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu -x > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
grep -E "packed N=|FAILED|Error" $OUT/pytest_gpu.log | head
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
bash scripts/gpu_ab.sh $OUT/ab "7cpa 3ce3" "nopk" 2
prof() {   # prof <tag> <config> <lib>
  DOCK_LIB=$3 timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_ls_adadelta -s 3 -c 1 \
      -o /tmp/p_$1 python bench.py --config $2 --steps 1 --warmup 0 --no-cpu --no-parts > $OUT/ncu_$1.log 2>&1
  python scripts/ncu_summary.py full /tmp/p_$1.ncu-rep > $OUT/full_$1.txt 2>&1
  ncu -i /tmp/p_$1.ncu-rep --page source --csv --print-source sass > $OUT/sass_$1.csv 2>&1
  gzip -f $OUT/sass_$1.csv
  python scripts/sass_blocks.py $OUT/sass_$1.csv.gz 30 > $OUT/blocks_$1.txt 2>&1
  head -30 $OUT/full_$1.txt; head -12 $OUT/blocks_$1.txt
}
prof 7cpa_pk 7cpa ""
