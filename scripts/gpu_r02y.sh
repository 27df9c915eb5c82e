#!/bin/bash
# round 2 pass y: packed tiles for the one-full-chunk shape too (33 <= N <= 48: 3ce3, HTS's
# mid-size ligands) -- the -m gpu suite, then A/B against DK_PACKED=0 (nopk)
set -u
OUT=gpurun_out/r02y; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
grep -E "FAILED|Error" $OUT/pytest_gpu.log | head
bash scripts/gpu_ab.sh $OUT/ab "3ce3 7cpa hts" "nopk" 2
