#!/bin/bash
# round 2 pass o: torsion-gradient lane blocks sized to the range lengths: parity + bench
set -u
OUT=gpurun_out/r02o; mkdir -p $OUT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ls_protocol.py -m gpu -q -x -rf -k "energy_gradient or deep_torsion or tail_schedules or max_size or large_ligand or adadelta or spec_style" > $OUT/pytest.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest.log
tail -3 $OUT/pytest.log
for rep in 1 2; do for C in 7cpa 3ce3; do
  timeout 300 python bench.py --config $C --steps 3 --warmup 2 --no-cpu --no-parts > $OUT/b_${C}_$rep.json 2>&1
  python -c "import json;d=json.loads(open('$OUT/b_${C}_$rep.json').read().strip().splitlines()[-1]);print('$C rep $rep', '%.4g'%d['value'])" 2>&1 | tail -1
done; done
