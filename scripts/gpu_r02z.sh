#!/bin/bash
# round 2 pass z: packed hybrid tail with paired transposed butterflies (default) vs one
# atom per butterfly (nopair); the -m gpu suite
set -u
OUT=gpurun_out/r02z; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa" "nopair" 3
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
grep -E "FAILED|Error" $OUT/pytest_gpu.log | head
