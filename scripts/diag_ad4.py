import sys; sys.path.insert(0, 'tests')
import numpy as np, oracle
from gen import config_inputs
from test_gpu_parity import near_reference_genotypes
import paper_2203_02096_b200 as dock
cfg, lig, grid = config_inputs('tiny')
for sf in (0, 1):
    d = dock.Docker.from_inputs(grid, lig, scoring=sf)
    P = oracle.Problem(grid, lig, sf={} if sf else None)
    X = near_reference_genotypes(grid, lig, d.T, 4, seed=31)
    for it in (1, 2):
        g, E, ev = d.ls_step(0, X, np.full(4, 1e30, np.float32), it)
        for i in range(2):
            x, Eo, _ = oracle.adadelta(P, oracle.params(), it, X[i], 1e30)
            print(sf, it, i, E[i], Eo, np.abs(g[i]-x).max())
    Eg, Gg, _ = d.eval(X, grad=True)
    for i in range(2):
        r = P.energy(X[i].astype(float))
        print('eval', Eg[i], r['E'], np.abs(Gg[i]-r['grad']).max(), np.abs(r['grad']).max())
