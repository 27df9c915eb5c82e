#!/bin/bash
# Source-level ncu profile of one kernel: per-CUDA-line and per-SASS-instruction execution
# counts (small CSVs; the .ncu-rep stays in /tmp).  Usage: bash scripts/gpu_srcprof.sh <tag> <config> <kernel-regex> [skip] [bench args]
set -u
TAG=$1; CFG=$2; KRE=$3; SKIP=${4:-5}; shift 4 || true
OUT=gpurun_out/$TAG; mkdir -p $OUT
[ -f paper_2203_02096_b200/libdock.so ] || python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:$KRE -s $SKIP -c 1 -o /tmp/sp_$CFG \
    python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu "$@" > $OUT/ncu_sp_$CFG.log 2>&1
ncu -i /tmp/sp_$CFG.ncu-rep --page source --csv --print-source cuda > $OUT/src_cuda_$CFG.csv 2>&1
ncu -i /tmp/sp_$CFG.ncu-rep --page source --csv --print-source sass > $OUT/src_sass_$CFG.csv 2>&1
python scripts/ncu_summary.py full /tmp/sp_$CFG.ncu-rep > $OUT/full_$CFG.txt 2>&1
rm -f /tmp/sp_$CFG.ncu-rep
ls -la $OUT
