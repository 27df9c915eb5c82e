#!/bin/bash
set -u
OUT=gpurun_out/ab7; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; tail -20 $OUT/build.log; exit 1; }
timeout 1200 python -m pytest tests -q -m gpu > $OUT/pytest.log 2>&1; echo "pytest rc=$?"; grep -E "passed|failed" $OUT/pytest.log | tail -3
for V in cur c7d78a6; do
  if [ $V = cur ]; then L=""; else L=build/variants/libdock_$V.so; fi
  for C in pm ps; do
    DOCK_LIB=$L timeout 600 python bench.py --config $C --runs 100 --sw-depth 1 --steps 2 --warmup 2 --no-cpu > $OUT/b_${C}_$V.json 2>$OUT/b_${C}_$V.err
    python -c "import json;d=json.loads(open('$OUT/b_${C}_$V.json').read().strip().splitlines()[-1]);print('$C runs 100 depth 1 $V', '%.4g'%d['value'], '%.1f ms'%d['ms_per_step'])" 2>/dev/null || { echo "$C $V failed"; tail -2 $OUT/b_${C}_$V.err; }
  done
done
for C in 1stp 3ce3 7cpa; do
  timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu > $OUT/b_$C.json 2>$OUT/b_$C.err
  python -c "import json;d=json.loads(open('$OUT/b_$C.json').read().strip().splitlines()[-1]);print('$C', '%.4g'%d['value'], '%.1f ms'%d['ms_per_step'])"
done
for C in pl pm; do for R in 10 100; do
  timeout 600 python bench.py --config $C --runs $R --steps 2 --warmup 2 --no-cpu > $OUT/b_${C}_r$R.json 2>$OUT/b_${C}_r$R.err
  python -c "import json;d=json.loads(open('$OUT/b_${C}_r$R.json').read().strip().splitlines()[-1]);print('$C runs $R auto', '%.4g'%d['value'], '%.1f ms'%d['ms_per_step'])"
done; done
