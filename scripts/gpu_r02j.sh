#!/bin/bash
# round 2 pass j: k_run_sw speculative GA: engine-equality + SW tests, A/B vs DK_RUNSW_SPEC=0 on 1stp / ps / pm
set -u
OUT=gpurun_out/r02j; mkdir -p $OUT
timeout 1200 python -m pytest tests -m gpu -q -x -rf -k "branches or cluster or sw_ or solis or screen or smoke or full_size or planted or statistics" > $OUT/pytest_sw.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_sw.log
tail -3 $OUT/pytest_sw.log
for rep in 1 2; do for C in 1stp; do for T in default nospec; do
  if [ $T = default ]; then L=""; else L=build/ab/libdock_$T.so; fi
  DOCK_LIB=$L timeout 300 python bench.py --config $C --steps 5 --warmup 2 --no-cpu --no-parts > $OUT/ab_${T}_${C}_$rep.json 2>&1
  python -c "import json;d=json.loads(open('$OUT/ab_${T}_${C}_$rep.json').read().strip().splitlines()[-1]);print('$C rep $rep $T', '%.4g'%d['value'], d['roofline']['share_of_step'])" 2>&1 | tail -1
done; done; done
for C in ps pm; do for T in default nospec; do
  if [ $T = default ]; then L=""; else L=build/ab/libdock_$T.so; fi
  DOCK_LIB=$L timeout 300 python bench.py --config $C --runs 10 --steps 3 --warmup 2 --no-cpu --no-parts > $OUT/ab_${T}_${C}.json 2>&1
  python -c "import json;d=json.loads(open('$OUT/ab_${T}_${C}.json').read().strip().splitlines()[-1]);print('$C $T', '%.4g'%d['value'])" 2>&1 | tail -1
done; done
