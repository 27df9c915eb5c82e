#!/bin/bash
# ncu evidence for profiles/: launch list of one bench step and a full capture of the
# dominant kernel.  Usage (on the GPU box): bash scripts/gpu_profile.sh <config> <kernel-regex> <tag>
set -u
CFG=${1:-1stp}; KRE=${2:-k_ls_sw}; TAG=${3:-r01}
mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file gpurun_out/launches_${CFG}_${TAG}.csv python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu \
    > gpurun_out/ncu_launch_${CFG}.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE} -s 20 -c 1 \
    -o gpurun_out/prof_${CFG}_${TAG} python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu \
    > gpurun_out/ncu_full_${CFG}.log 2>&1
echo "profile done $CFG $KRE"
