#!/bin/bash
# round 2 pass h: hybrid tail (chunks x tail broadcast + segment rounds) vs round-1 broadcast, tail parity
set -u
OUT=gpurun_out/r02h; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -rf -k "tail_schedules or energy_gradient_pose" > $OUT/pytest_tail.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_tail.log
tail -3 $OUT/pytest_tail.log
for rep in 1 2; do for C in 7cpa pm; do for T in default bcast1; do
  if [ $T = default ]; then E=""; else E=$T; fi
  DOCK_TAIL=$E timeout 300 python bench.py --config $C --steps 3 --warmup 2 --no-cpu --no-parts > $OUT/ab_${T}_${C}_$rep.json 2>&1
  python -c "import json;d=json.loads(open('$OUT/ab_${T}_${C}_$rep.json').read().strip().splitlines()[-1]);print('$C rep $rep $T', '%.4g'%d['value'])" 2>&1 | tail -1
done; done; done
