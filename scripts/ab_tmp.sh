#!/bin/bash
set -u
OUT=gpurun_out/ab1; mkdir -p $OUT
python -c "import __graft_entry__ as g; g.build()" > $OUT/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], d.get('score_evals_per_s'))" 2>/dev/null || tail -3 ${1%.json}.err; }
for V in cur f76266f ffe2d77 bbdf148 b3b4a64 987caa8; do
  if [ $V = cur ]; then L=""; else L=build/variants/libdock_$V.so; fi
  DOCK_LIB=$L timeout 600 python bench.py --config hts --n-ligs 256 --steps 2 --warmup 2 --no-cpu > $OUT/hts_$V.json 2>$OUT/hts_$V.err; j $OUT/hts_$V.json
done
for V in cur w32; do
  if [ $V = cur ]; then L=""; else L=build/variants/libdock_$V.so; fi
  DOCK_LIB=$L timeout 600 python bench.py --config 1stp --steps 3 --warmup 3 --no-cpu > $OUT/1stp_$V.json 2>$OUT/1stp_$V.err; j $OUT/1stp_$V.json
done
