#!/bin/bash
set -u
OUT=gpurun_out/r01c; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
timeout 900 python -m pytest tests -q -m gpu > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -8 $OUT/pytest_gpu.log
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);r=d.get('roofline') or {};print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], r.get('avg_launch_ms'), r.get('frac'))"; }
for D in 1 2 3 0; do
  timeout 600 python bench.py --config 1stp --steps 3 --warmup 3 --no-cpu --sw-depth $D > $OUT/b_1stp_d$D.json 2>$OUT/b_1stp_d$D.err; j $OUT/b_1stp_d$D.json
done
for V in default fdiv ada3; do
  if [ $V = default ]; then L=""; else L=build/variants/libdock_$V.so; fi
  DOCK_LIB=$L timeout 600 python bench.py --config 7cpa --steps 2 --warmup 3 --no-cpu > $OUT/b_7cpa_$V.json 2>$OUT/b_7cpa_$V.err; j $OUT/b_7cpa_$V.json
  DOCK_LIB=$L timeout 600 python bench.py --config 3ce3 --steps 3 --warmup 3 --no-cpu > $OUT/b_3ce3_$V.json 2>$OUT/b_3ce3_$V.err; j $OUT/b_3ce3_$V.json
done
timeout 900 python bench.py --config hts --n-ligs 64 --steps 2 --warmup 3 > $OUT/b_hts.json 2>$OUT/b_hts.err; echo "hts rc=$?"; tail -c 1500 $OUT/b_hts.json; tail -3 $OUT/b_hts.err
