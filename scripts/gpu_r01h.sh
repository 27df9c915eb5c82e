#!/bin/bash
set -u
OUT=gpurun_out/r01h; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu.log
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);r=d.get('roofline') or {};print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], r.get('avg_launch_ms'), r.get('frac'))"; }
DOCK_TRACE=1 timeout 600 python scripts/e2e_probe.py 1stp > $OUT/e2e_1stp.log 2>&1; grep -E "rep|ctx\." $OUT/e2e_1stp.log | tail -16
for C in 1stp 3ce3 7cpa tiny; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu > $OUT/b_$C.json 2>$OUT/b_$C.err; j $OUT/b_$C.json
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bench_part -s 2 -c 1 -o gpurun_out/prof_micro_intra_7cpa_r01h python bench.py --micro --config 7cpa --steps 1 --micro-iters 5 > $OUT/ncu_micro.log 2>&1; tail -1 $OUT/ncu_micro.log
