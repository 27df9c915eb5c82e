#!/bin/bash
# round 2 pass k: ADADELTA lockstep vs run branches when one GPU holds few runs (the R split at 2/4/8 GPUs)
set -u
OUT=gpurun_out/r02k; mkdir -p $OUT
for R in 13 25 50 100; do for B in 1 2; do
  timeout 300 python bench.py --config 7cpa --runs $R --run-branches $B --steps 3 --warmup 2 --no-cpu --no-parts > $OUT/b_r${R}_b$B.json 2>&1
  python -c "import json;d=json.loads(open('$OUT/b_r${R}_b$B.json').read().strip().splitlines()[-1]);print('7cpa runs $R branches $B', '%.4g'%d['value'], d['ms_per_step'])" 2>&1 | tail -1
done; done
