"""Diagnostics: print the worst eval / ADADELTA mismatches vs the oracle (GPU box)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import paper_2203_02096_b200 as dock
from gen import config_inputs, random_genotypes

for name in sys.argv[1:] or ["1stp", "3ce3"]:
    cfg, lig, grid = config_inputs(name)
    d = dock.Docker.from_inputs(grid, lig)
    P = oracle.Problem(grid, lig)
    X = random_genotypes(grid, d.T, 200, seed=7, frac_out=0.05)
    E, Gd, xyz = d.eval(X, grad=True, xyz=True)
    E0, _, _ = d.eval(X)
    nbad = 0
    for i in range(200):
        ref = P.energy(X[i].astype(np.float64))
        fm, cm = P.margins(ref["xyz"])
        dx = np.abs(xyz[i] - ref["xyz"]).max()
        de = abs(E[i] - ref["E"]); de0 = abs(E0[i] - ref["E"])
        dg = np.abs(Gd[i] - ref["grad"]).max() / max(1, np.abs(ref["grad"]).max())
        if dx > 1e-4 or de > max(1e-3, 1e-4 * abs(ref["E"])) or de0 > max(1e-3, 1e-4*abs(ref["E"])) or dg > 1e-3:
            nbad += 1
            if nbad <= 6:
                print(name, i, "dx %.2e" % dx, "E %.6g ref %.6g E0 %.6g" % (E[i], ref["E"], E0[i]),
                      "inter %.6g intra %.6g" % (ref["inter"], ref["intra"]), "dg %.2e" % dg, "fm %.1e cm %.1e" % (fm, cm))
                j = np.argmax(np.abs(Gd[i] - ref["grad"])); print("   grad j", j, Gd[i][j], ref["grad"][j])
    print(name, "bad", nbad, "of 200")
    # ADADELTA
    X = random_genotypes(grid, d.T, 16, seed=31, frac_out=0.0, shrink=0.2)
    for iters in (1, 2, 5):
        g, Eg, ev = d.ls_step(0, X, np.full(16, 1e30, np.float32), iters)
        pp = oracle.params()
        for i in range(4):
            x, Eo, evo = oracle.adadelta(P, pp, iters, X[i], 1e30)
            print(" ada", iters, i, "E %.6g ref %.6g" % (Eg[i], Eo), "dgenes %.2e" % np.abs(g[i] - x).max())
