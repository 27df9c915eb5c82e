#!/bin/bash
# GPU pass: build, the -m gpu suite, smoke, and short bench lines for the three single-ligand configs.
set -u
OUT=gpurun_out/${1:-tests}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error" $OUT/pytest_gpu.log | tail -8
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 $OUT/smoke.log
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);r=d.get('roofline') or {};print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], r.get('avg_launch_ms'), r.get('frac'))"; }
for C in ${CFGS:-1stp 3ce3 7cpa}; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu > $OUT/b_$C.json 2>$OUT/b_$C.err; j $OUT/b_$C.json
done
