#!/bin/bash
# round 2 pass za: four tail atoms per transposed butterfly (quad) vs two (default);
# the -m gpu suite
set -u
OUT=gpurun_out/r02za; mkdir -p $OUT
bash scripts/gpu_ab.sh $OUT/ab "7cpa" "quad" 3
DOCK_LIB=build/ab/libdock_quad.so timeout 1200 python -m pytest tests/test_gpu_parity.py -q -m gpu -k "packed or tail or energy_gradient" > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu.log
grep -E "FAILED|Error" $OUT/pytest_gpu.log | head
