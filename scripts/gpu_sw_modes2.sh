#!/bin/bash
OUT=gpurun_out/swmodes2; mkdir -p $OUT
[ -f paper_2203_02096_b200/libdock.so ] || python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
python - <<'PY' 2>&1 | tee $OUT/modes.txt
import sys, time, os
sys.path.insert(0, ".")
import torch
import paper_2203_02096_b200 as dock
from gen import config_inputs
for name, runs in [("ps", 100), ("pm", 100), ("ps", 40), ("1stp", 50)]:
    cfg, lig, grid = config_inputs(name)
    for mode, env in ((2, None), (3, "1")):
        if env: os.environ["DOCK_RUNSW_ANY"] = env  # (round 1; now the -DDK_RUNSW_ANY=1 build variant)
        else: os.environ.pop("DOCK_RUNSW_ANY", None)
        d = dock.Docker.from_inputs(grid, lig, ls_method=1, ls_rate=cfg.ls_rate, ls_max_iters=cfg.ls_iters, run_branches=mode)
        budget = cfg.max_evals if name == "1stp" else 1_000_000
        d.run(cfg.pop, runs, budget // 10, 1, xyz=False)
        torch.cuda.synchronize(); t0 = time.perf_counter()
        r = d.run(cfg.pop, runs, budget, 42, xyz=False)
        dt = time.perf_counter() - t0
        print(f"{name} runs {runs} mode {mode} any={env}: {r['evals'].sum() / dt:.4g} evals/s, {1e3 * dt:.1f} ms", flush=True)
        d.close()
PY
