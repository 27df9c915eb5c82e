#!/bin/bash
set -u
OUT=gpurun_out/ab2; mkdir -p $OUT
bash scripts/gpu_tests.sh ab2t
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'], d.get('score_evals_per_s'))" 2>/dev/null || tail -3 ${1%.json}.err; }
for V in cur f76266f; do
  if [ $V = cur ]; then L=""; else L=build/variants/libdock_$V.so; fi
  DOCK_LIB=$L timeout 600 python bench.py --config hts --n-ligs 256 --steps 2 --warmup 2 --no-cpu > $OUT/hts_$V.json 2>$OUT/hts_$V.err; j $OUT/hts_$V.json
done
