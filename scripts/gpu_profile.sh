#!/bin/bash
# ncu evidence for profiles/: launch list of one bench step and a full capture of the
# dominant kernel, summarised on the box (the .ncu-rep stays in /tmp: gpurun copies back
# at most 64 MiB).  Usage (on the GPU box): bash scripts/gpu_profile.sh <config> <kernel-regex> <tag> [bench args]
set -u
CFG=${1:-1stp}; KRE=${2:-k_ls_sw}; TAG=${3:-r01}; shift 3 || true
OUT=gpurun_out/$TAG
mkdir -p $OUT
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
    --log-file $OUT/launches_${CFG}.csv python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu "$@" \
    > $OUT/ncu_launch_${CFG}.log 2>&1
python scripts/ncu_summary.py launches $OUT/launches_${CFG}.csv > $OUT/launch_share_${CFG}.txt 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:${KRE} -s ${SKIP:-20} -c 1 \
    -o /tmp/prof_${CFG}_${TAG} python bench.py --config $CFG --steps 1 --warmup 0 --no-cpu "$@" \
    > $OUT/ncu_full_${CFG}.log 2>&1
python scripts/ncu_summary.py full /tmp/prof_${CFG}_${TAG}.ncu-rep > $OUT/full_ls_${CFG}.txt 2>&1
rm -f /tmp/prof_${CFG}_${TAG}.ncu-rep
echo "profile done $CFG $KRE: $(grep -m1 duration $OUT/full_ls_${CFG}.txt)"
