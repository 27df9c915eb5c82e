#!/bin/bash
OUT=gpurun_out/abd3; mkdir -p $OUT
[ -f paper_2203_02096_b200/libdock.so ] || python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python - <<'PY' 2>&1 | tee $OUT/d3.txt
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2203_02096_b200 as dock
from gen import config_inputs
for name, runs in [("1stp", 20), ("ps", 10), ("pm", 10), ("1stp", 5)]:
    cfg, lig, grid = config_inputs(name)
    res = {}
    for depth in (2, 3):
        d = dock.Docker.from_inputs(grid, lig, ls_method=1, ls_rate=cfg.ls_rate, ls_max_iters=cfg.ls_iters, run_branches=3, sw_depth=depth)
        budget = cfg.max_evals if name == "1stp" else 1_000_000
        d.run(cfg.pop, runs, budget // 10, 1, xyz=False)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = d.run(cfg.pop, runs, budget, 42, xyz=False)
        dt = time.perf_counter() - t0
        res[depth] = r
        print(f"{name} runs {runs} depth {depth}: {r['evals'].sum() / dt:.4g} evals/s, {1e3 * dt:.1f} ms", flush=True)
        d.close()
    print("  identical:", all(np.array_equal(res[2][k], res[3][k]) for k in ("best_E", "best_genes", "evals")), flush=True)
PY
