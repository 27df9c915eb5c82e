"""Where does the end-to-end (host API) time of one docking job go? dock_init / dock_run_ex /
dock_free wall times for a config, repeated (first repetition includes module loading)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2203_02096_b200 as dock
from gen import config_inputs

name = sys.argv[1] if len(sys.argv) > 1 else "1stp"
cfg, lig, grid = config_inputs(name)
tp, roles = grid.type_params()
for rep in range(4):
    t0 = time.perf_counter()
    d = dock.Docker(grid.maps, grid.n, grid.spacing, grid.origin, tp, roles, lig.types, lig.charges, lig.xyz,
                    lig.bonds, lig.rotatable, ls_method=cfg.ls_method, ls_rate=cfg.ls_rate, ls_max_iters=cfg.ls_iters)
    t1 = time.perf_counter()
    r = d.run(cfg.pop, cfg.runs, cfg.max_evals, 42, xyz=True)
    t2 = time.perf_counter()
    d.close()
    t3 = time.perf_counter()
    ev = int(r["evals"].sum())
    print(f"{name} rep {rep}: init {1e3*(t1-t0):.1f} ms, run {1e3*(t2-t1):.1f} ms, free {1e3*(t3-t2):.1f} ms, "
          f"evals {ev} -> {ev/(t3-t0):.4g} evals/s e2e, {ev/(t2-t1):.4g} run-only", flush=True)
