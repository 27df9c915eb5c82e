#!/bin/bash
set -u
OUT=gpurun_out/r01o; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" $OUT/pytest_gpu.log | tail -3
for R in 10 100; do
  timeout 600 python bench.py --config pl --runs $R --steps 2 --warmup 2 --no-cpu > $OUT/b_pl_r$R.json 2>$OUT/b_pl_r$R.err
  python -c "import json;d=json.loads(open('$OUT/b_pl_r$R.json').read().strip().splitlines()[-1]);print('pl runs $R auto', '%.4g'%d['value'], '%.1f ms'%d['ms_per_step'])"
done
bash scripts/gpu_round.sh r01o
