#!/bin/bash
# round 2 pass zb: back-projection sums by one transposed reduction (default) vs nobpt, and
# the torsion range walk unrolled by 2 (default) vs walk1; the -m gpu suite
set -u
OUT=gpurun_out/r02zb; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa 3ce3" "nobpt walk1" 2
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
grep -E "FAILED|Error" $OUT/pytest_gpu.log | head
