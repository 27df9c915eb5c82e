#!/bin/bash
# round 2 pass l: ADADELTA auto branches (few runs per GPU): full GPU suite, 7cpa 13/100 runs, HTS auto vs lockstep
set -u
OUT=gpurun_out/r02l; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -3 $OUT/pytest_gpu.log
for R in 13 100; do
  timeout 300 python bench.py --config 7cpa --runs $R --steps 3 --warmup 2 --no-cpu --no-parts > $OUT/b_r$R.json 2>&1
  python -c "import json;d=json.loads(open('$OUT/b_r$R.json').read().strip().splitlines()[-1]);print('7cpa runs $R auto', '%.4g'%d['value'], d['roofline']['engine'])" 2>&1 | tail -1
done
for B in 0 1; do
  timeout 600 python bench.py --config hts --n-ligs 256 --steps 2 --warmup 1 --no-cpu --run-branches $B > $OUT/hts_b$B.json 2>&1
  python -c "import json;d=json.loads(open('$OUT/hts_b$B.json').read().strip().splitlines()[-1]);print('hts run_branches $B', '%.4g'%d['value'])" 2>&1 | tail -1
done
