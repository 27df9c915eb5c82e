#!/bin/bash
# Multi-rank bench path on a 1-GPU box: torchrun 2 ranks, gloo over CPU tensors, both ranks on
# GPU 0 (BENCH_DIST_TEST=1, test-only mode of bench.py); checks sharding, barriers,
# max-over-ranks and the final gathers.
set -u
OUT=gpurun_out/${1:-dist}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
BENCH_DIST_TEST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --config 1stp --steps 2 --warmup 3 > $OUT/b_3ce3_2r.json 2> $OUT/b_3ce3_2r.err; echo "3ce3 2 ranks rc=$?"; tail -c 700 $OUT/b_3ce3_2r.json; tail -3 $OUT/b_3ce3_2r.err
BENCH_DIST_TEST=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config hts --n-ligs 32 --steps 1 --warmup 3 > $OUT/b_hts_2r.json 2> $OUT/b_hts_2r.err; echo "hts 2 ranks rc=$?"; tail -c 500 $OUT/b_hts_2r.json; tail -3 $OUT/b_hts_2r.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --config 1stp --steps 1 --warmup 1 > $OUT/ref_2r.json 2> $OUT/ref_2r.err; echo "reference 2 ranks rc=$?"; tail -c 300 $OUT/ref_2r.json
