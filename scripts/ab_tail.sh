#!/bin/bash
# A/B of the gradient-tile tail schedules (DOCK_TAIL=seg|other) on ADADELTA configs.
OUT=gpurun_out/abtail; mkdir -p $OUT
[ -f paper_2203_02096_b200/libdock.so ] || python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
for C in 3ce3 7cpa; do for M in seg bcast; do
  DOCK_TAIL=$M timeout 600 python bench.py --config $C --steps 3 --warmup 2 --no-cpu > $OUT/b_${C}_$M.json 2>&1
  python -c "import json;d=json.loads(open('$OUT/b_${C}_$M.json').read().strip().splitlines()[-1]);print('$C $M', '%.4g'%d['value'])"
done; done
