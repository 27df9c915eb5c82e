#!/bin/bash
# round 2 pass zf: packed tile (0,0) for the one-chunk shape (33 <= N <= 48, 3ce3) --
# the -m gpu suite, then A/B against DK_PACKED=0 on 3ce3, HTS and 7cpa
set -u
OUT=gpurun_out/r02zf; mkdir -p $OUT
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
grep -E "FAILED|Error" $OUT/pytest_gpu.log | head
bash scripts/gpu_ab.sh $OUT/ab "3ce3 hts 7cpa" "nopk" 2
