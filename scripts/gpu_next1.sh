#!/bin/bash
# NEXT-1: the paper's input shapes PS/PM/PL x Solis-Wets speculation depth
# (lane groups per individual: depth 1 = 2, depth 2 = 8, depth 3 = 26) x nruns {10, 100}.
set -u
OUT=gpurun_out/${1:-next1}; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
timeout 900 python -m pytest tests -q -m gpu -k "parity and (pm or pl)" > $OUT/pytest_next1.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_next1.log
for C in ps pm pl; do for R in 10 100; do for D in 1 2 3; do
  timeout 600 python bench.py --config $C --runs $R --sw-depth $D --steps 2 --warmup 2 --no-cpu > $OUT/b_${C}_r${R}_d${D}.json 2>$OUT/b_${C}_r${R}_d${D}.err
  python -c "import json;d=json.loads(open('$OUT/b_${C}_r${R}_d${D}.json').read().strip().splitlines()[-1]);print('$C runs $R depth $D', '%.4g'%d['value'], '%.1f ms'%d['ms_per_step'])" 2>/dev/null || { echo "$C $R $D failed"; tail -2 $OUT/b_${C}_r${R}_d${D}.err; }
done; done; done
