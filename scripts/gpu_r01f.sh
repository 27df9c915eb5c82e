#!/bin/bash
set -u
OUT=gpurun_out/r01f; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu.log
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);r=d.get('roofline') or {};print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], r.get('avg_launch_ms'), r.get('frac'))"; }
DOCK_TRACE=1 timeout 600 python scripts/e2e_probe.py 1stp > $OUT/e2e_1stp.log 2>&1; grep -v "^\[dock\] run.graph" $OUT/e2e_1stp.log | tail -22
for V in default tab; do
  if [ $V = default ]; then L=""; else L=build/variants/libdock_$V.so; fi
  for C in 3ce3 7cpa; do
    DOCK_LIB=$L timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu > $OUT/b_${C}_$V.json 2>$OUT/b_${C}_$V.err; j $OUT/b_${C}_$V.json
  done
done
for D in 2 3; do
  timeout 600 python bench.py --config 1stp --steps 3 --warmup 3 --no-cpu --sw-depth $D > $OUT/b_1stp_d$D.json 2>$OUT/b_1stp_d$D.err; j $OUT/b_1stp_d$D.json
done
