#!/bin/bash
set -u
OUT=gpurun_out/r01e; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 $OUT/pytest_gpu.log
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);r=d.get('roofline') or {};print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], r.get('avg_launch_ms'), r.get('frac'))"; }
timeout 600 python scripts/e2e_probe.py 1stp > $OUT/e2e_1stp.log 2>&1; cat $OUT/e2e_1stp.log
for C in 7cpa 3ce3 1stp; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu > $OUT/b_$C.json 2>$OUT/b_$C.err; j $OUT/b_$C.json
done
