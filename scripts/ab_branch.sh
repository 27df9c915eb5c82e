#!/bin/bash
OUT=gpurun_out/abbr; mkdir -p $OUT
[ -f paper_2203_02096_b200/libdock.so ] || python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python - <<'PY'
import json, time, sys
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2203_02096_b200 as dock
from gen import config_inputs
for name in ["1stp", "ps"]:
    cfg, lig, grid = config_inputs(name)
    for rb in (1, 2):
        for K in (16, 32, 64):
            d = dock.Docker.from_inputs(grid, lig, ls_method=cfg.ls_method, ls_rate=cfg.ls_rate,
                                        ls_max_iters=cfg.ls_iters, run_branches=rb, gens_per_graph=K)
            d.run(cfg.pop, cfg.runs, cfg.max_evals // 10, 1, xyz=False)
            torch.cuda.synchronize(); t0 = time.perf_counter()
            r = d.run(cfg.pop, cfg.runs, cfg.max_evals, 42, xyz=False)
            dt = time.perf_counter() - t0
            print(name, "branches" if rb == 2 else "lockstep", "K", K, "%.4g evals/s" % (r["evals"].sum() / dt), "%.1f ms" % (1e3 * dt), flush=True)
            d.close()
PY
