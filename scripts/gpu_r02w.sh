#!/bin/bash
# round 2 pass w: packed-loop software pipeline (default, unroll 2) vs nopf / pf16, and the
# branch-free two-pass grid gathers (default) vs nobf; then the -m gpu suite
set -u
OUT=gpurun_out/r02w; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa 3ce3" "nopf pf16 nobf" 2
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
grep -E "FAILED|Error" $OUT/pytest_gpu.log | head
