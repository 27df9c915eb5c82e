#!/bin/bash
# round 2 pass zh: the H-bond segmented scan bounded by the longest segment (default) vs all
# five levels (hbfull); the -m gpu suite
set -u
OUT=gpurun_out/r02zh; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa" "hbfull" 3
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_gpu.log
grep -E "FAILED|Error" $OUT/pytest_gpu.log | head
