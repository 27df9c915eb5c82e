#!/bin/bash
# round 2 pass e: folded D5 slot constants, torsion-gradient pieces, grouped-broadcast tail:
# parity (full GPU suite) + bench 7cpa / 3ce3 / 1stp
set -u
OUT=gpurun_out/r02e; mkdir -p $OUT
timeout 1500 python -m pytest tests -m gpu -q -x -rf > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
tail -5 $OUT/pytest_gpu.log
for C in 7cpa 3ce3 1stp; do
  timeout 300 python bench.py --config $C --steps 3 --warmup 3 --no-cpu > $OUT/bench_$C.json 2> $OUT/bench_$C.err
  python -c "import json;d=json.loads(open('$OUT/bench_$C.json').read().strip().splitlines()[-1]);print('$C', '%.4g'%d['value'], d['roofline']['frac'])"
done
DOCK_TAIL=bcast1 timeout 300 python bench.py --config 7cpa --steps 3 --warmup 3 --no-cpu > $OUT/bench_7cpa_bcast1.json 2>&1
python -c "import json;d=json.loads(open('$OUT/bench_7cpa_bcast1.json').read().strip().splitlines()[-1]);print('7cpa bcast1', '%.4g'%d['value'])"
