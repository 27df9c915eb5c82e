#!/bin/bash
# round 2 pass c: full GPU suite after the parity-protocol hooks and the kernels.cu split; bench 7cpa + 1stp
set -u
OUT=gpurun_out/r02c; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -s -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
grep -E "SW free|ADADELTA free|ADADELTA trajectory|passed|failed|FAILED" $OUT/pytest_gpu.log | tail -40
timeout 300 python bench.py --steps 3 --warmup 3 --no-cpu > $OUT/bench_7cpa.json 2> $OUT/bench_7cpa.err; tail -c 300 $OUT/bench_7cpa.json
timeout 300 python bench.py --config 1stp --steps 5 --warmup 3 --no-cpu > $OUT/bench_1stp.json 2> $OUT/bench_1stp.err; tail -c 300 $OUT/bench_1stp.json
