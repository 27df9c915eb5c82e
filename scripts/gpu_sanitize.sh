#!/bin/bash
# compute-sanitizer racecheck / memcheck over the packed gradient path (7cpa: k_eval PK and a
# short ADADELTA run) and the scalar path (3ce3): shared-memory hazards of the scratch reuse
set -u
OUT=gpurun_out/san; mkdir -p $OUT
cat > /tmp/san.py <<'PY'
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2203_02096_b200 as dock
from gen import config_inputs, random_genotypes
for name in sys.argv[1:]:
    cfg, lig, grid = config_inputs(name)
    d = dock.Docker.from_inputs(grid, lig, ls_method=0, ls_rate=1.0, ls_max_iters=20)
    X = random_genotypes(grid, d.T, 64, seed=3)
    E, G, _ = d.eval(X, grad=True, xyz=True)
    r = d.run(32, 2, 32 * 60, 7)
    print(name, d.tile_schedule, float(E.mean()), r["best_E"])
PY
for tool in racecheck memcheck; do
  X=""; [ $tool = racecheck ] && X="--racecheck-report hazard"
  timeout 1200 compute-sanitizer --tool $tool $X python /tmp/san.py 7cpa 3ce3 > $OUT/$tool.log 2>&1
  echo "$tool rc=$?"; tail -4 $OUT/$tool.log
done
