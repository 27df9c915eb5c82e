#!/bin/bash
# Solis-Wets engines on the paper's shapes: lockstep (1), branches (2), persistent clusters (3).
OUT=gpurun_out/swmodes; mkdir -p $OUT
[ -f paper_2203_02096_b200/libdock.so ] || python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python - <<'PY' 2>&1 | tee $OUT/modes.txt
import sys, time
sys.path.insert(0, ".")
import torch
import paper_2203_02096_b200 as dock
from gen import config_inputs
for name, runs in [("1stp", 20), ("ps", 10), ("ps", 100), ("pm", 10), ("pm", 100), ("pl", 10)]:
    cfg, lig, grid = config_inputs(name)
    for mode in (1, 2, 3):
        d = dock.Docker.from_inputs(grid, lig, ls_method=1, ls_rate=cfg.ls_rate, ls_max_iters=cfg.ls_iters,
                                    run_branches=mode)
        budget = cfg.max_evals if name == "1stp" else 1_000_000
        d.run(cfg.pop, runs, budget // 10, 1, xyz=False)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = d.run(cfg.pop, runs, budget, 42, xyz=False)
        dt = time.perf_counter() - t0
        print(f"{name} runs {runs} mode {mode} (branches {d.run_branches}): {r['evals'].sum() / dt:.4g} evals/s, {1e3 * dt:.1f} ms", flush=True)
        d.close()
PY
