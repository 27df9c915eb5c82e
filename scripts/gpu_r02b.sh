#!/bin/bash
# round 2 pass b: the at-pose parity, generation 0, SW fed / free-run and ADADELTA protocol tests
set -u
OUT=gpurun_out/r02b; mkdir -p $OUT
timeout 1200 python -m pytest tests/test_gpu_ls_protocol.py tests/test_gpu_parity.py tests/test_gpu_ad4.py -m gpu -q -s -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
grep -E "^parity|SW free|ADADELTA free|passed|failed|Error|assert" $OUT/pytest_gpu.log | tail -80
