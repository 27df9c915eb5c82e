#!/bin/bash
# round 2 pass ze: packed tiles also for 49 <= N <= 64 (two chunks, the second padded and
# rotated) -- the -m gpu suite, then A/B against DK_PACKED=0 on the HTS sample and 7cpa
set -u
OUT=gpurun_out/r02ze; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
grep -E "FAILED|Error" $OUT/pytest_gpu.log | head
bash scripts/gpu_ab.sh $OUT/ab "hts 7cpa" "nopk" 3
