#!/bin/bash
set -u
OUT=gpurun_out/r01i; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);r=d.get('roofline') or {};print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], 'e2e %.4g'%d['e2e']['value'], r.get('avg_launch_ms'), r.get('frac'))"; }
timeout 600 python bench.py --config 1stp > $OUT/b_1stp.json 2>$OUT/b_1stp.err; j $OUT/b_1stp.json
for S in 4 8 16; do
  timeout 600 python bench.py --config hts --n-ligs 128 --steps 2 --warmup 3 --no-cpu --slots $S > $OUT/b_hts_s$S.json 2>$OUT/b_hts_s$S.err; j $OUT/b_hts_s$S.json
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ls_adadelta -s 5 -c 1 -o gpurun_out/prof_7cpa_r01i python bench.py --config 7cpa --steps 1 --warmup 0 --no-cpu > $OUT/ncu_7cpa.log 2>&1; tail -1 $OUT/ncu_7cpa.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ls_adadelta -s 5 -c 1 -o gpurun_out/prof_3ce3_r01i python bench.py --config 3ce3 --steps 1 --warmup 0 --no-cpu > $OUT/ncu_3ce3.log 2>&1; tail -1 $OUT/ncu_3ce3.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_bench_part -s 3 -c 1 -o gpurun_out/prof_micro_intra_7cpa_r01i python bench.py --micro --config 7cpa --steps 1 --micro-iters 5 > $OUT/ncu_micro.log 2>&1; tail -1 $OUT/ncu_micro.log
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_ls_sw -s 20 -c 1 -o gpurun_out/prof_1stp_r01i python bench.py --config 1stp --steps 1 --warmup 0 --no-cpu > $OUT/ncu_1stp.log 2>&1; tail -1 $OUT/ncu_1stp.log
