#!/bin/bash
set -u
OUT=gpurun_out/ab4; mkdir -p $OUT
bash scripts/gpu_tests.sh ab4t
j() { python -c "import json,sys;d=json.loads(open('$1').read().strip().splitlines()[-1]);print('$1', '%.4g'%d['value'], '%.1f'%d['ms_per_step'])" 2>/dev/null || tail -3 ${1%.json}.err; }
for V in nowalk walk5; do
  for C in 1stp 3ce3 7cpa; do
    DOCK_LIB=build/variants/libdock_$V.so timeout 600 python bench.py --config $C --steps 3 --warmup 3 --no-cpu > $OUT/${C}_$V.json 2>$OUT/${C}_$V.err; j $OUT/${C}_$V.json
  done
done
python - <<'PY'
import sys; sys.path.insert(0,'.')
import numpy as np
import oracle
from gen import config_inputs
for n in ['tiny','1stp','3ce3','7cpa','ps','pm','pl']:
    cfg,lig,grid=config_inputs(n); P=oracle.Problem(grid,lig)
    print(n, 'torsions', len(P.topo['tor_a']))
PY
