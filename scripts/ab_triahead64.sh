#!/bin/bash
# A/B: the Solis-Wets deviate window of the tree chain (DK_TRI_AHEAD), default 32 vs 64.
# Cluster-engine parity tests first, then alternating bench lines on the cluster-eligible shapes.
set -u
OUT=gpurun_out/abta64; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -30 $OUT/build.log; exit 1; }
python scripts/variants.py ta64=DK_TRI_AHEAD=64 > $OUT/build_var.log 2>&1 || { echo VARIANT BUILD FAILED; tail -30 $OUT/build_var.log; exit 1; }
for V in default ta64; do
  if [ $V = default ]; then L=""; else L=build/variants/libdock_$V.so; fi
  DOCK_LIB=$L timeout 900 python -m pytest tests -q -m gpu -k "run_branches or cluster or smoke or screen" > $OUT/pytest_cluster_$V.log 2>&1
  echo "pytest $V rc=$?"; grep -E "passed|failed|Error" $OUT/pytest_cluster_$V.log | tail -5
done
for rep in 1 2; do
  for C in "1stp" "ps --runs 10"; do
    T=$(echo $C | tr -d ' -')
    for V in default ta64; do
      if [ $V = default ]; then L=""; else L=build/variants/libdock_$V.so; fi
      DOCK_LIB=$L timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu > $OUT/b_${T}_${V}_$rep.json 2>$OUT/b_${T}_${V}_$rep.err
      python -c "import json;d=json.loads(open('$OUT/b_${T}_${V}_$rep.json').read().strip().splitlines()[-1]);r=d['roofline'];print('$T $V $rep', '%.4g'%d['value'], r.get('engine'), '%.3f'%r['share_of_step'])"
    done
  done
done
