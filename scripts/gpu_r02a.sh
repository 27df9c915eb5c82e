#!/bin/bash
# round 2, first pass: pipe microbenchmark, GPU tests, default bench line (7cpa)
set -u
OUT=gpurun_out/r02a; mkdir -p $OUT
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/ubench scripts/ubench_pipes.cu && timeout 120 /tmp/ubench > $OUT/ubench_pipes.txt 2>&1
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv >> $OUT/ubench_pipes.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
timeout 600 python bench.py --steps 5 --warmup 3 > $OUT/bench_7cpa.json 2> $OUT/bench_7cpa.err; tail -c 600 $OUT/bench_7cpa.json
