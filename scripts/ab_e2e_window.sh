#!/bin/bash
# e2e (host API) of 1stp with deviate window 32 (default) vs 16: is the r01v/r01w e2e drop the window or the box?
set -u
OUT=gpurun_out/abe2e; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
python scripts/variants.py ta16=DK_TRI_AHEAD=16 > $OUT/build_var.log 2>&1 || { echo VARIANT BUILD FAILED; exit 1; }
for rep in 1 2; do for V in default ta16; do
  if [ $V = default ]; then L=""; else L=build/variants/libdock_$V.so; fi
  DOCK_LIB=$L timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > $OUT/b_${V}_$rep.json 2>$OUT/b_${V}_$rep.err
  python -c "import json;d=json.loads(open('$OUT/b_${V}_$rep.json').read().strip().splitlines()[-1]);print('$V $rep', '%.4g'%d['value'], 'e2e %.4g'%d['e2e']['value'])"
done; done
