#!/bin/bash
# round 2 pass v: packed tiles, (a) and (b) fused into one loop (default, unroll 2) against
# fuse1 (fused, unroll 1) and nofuse (two loops, unroll 2); then the -m gpu suite
set -u
OUT=gpurun_out/r02v; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa" "fuse1 nofuse" 2
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
grep -E "FAILED|Error" $OUT/pytest_gpu.log | head
grep -E "parity packed" $OUT/pytest_gpu.log | head -8
