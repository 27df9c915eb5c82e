#!/bin/bash
# NEXT-2 GPU pass: the whole -m gpu suite (D5 + AD4), then D5 and AD4 bench lines.
set -u
OUT=gpurun_out/${1:-ad4}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 1500 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed|Error" $OUT/pytest_gpu.log | tail -8
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);r=d.get('roofline') or {};print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], r.get('avg_launch_ms'), r.get('frac'))"; }
for C in ${CFGS:-1stp 3ce3 7cpa}; do
  for S in d5 ad4; do
    timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu --scoring $S > $OUT/b_${C}_$S.json 2>$OUT/b_${C}_$S.err; j $OUT/b_${C}_$S.json
  done
done
