"""Pins for the oracle's D5 intramolecular energy."""
import math

import numpy as np
import pytest

from gen import constant_grid, make_ligand
from gen.synth import TYPE_TABLE
import oracle


class _Lig:
    pass


def two_atoms(names, q=(0.0, 0.0), sep=6):
    """Two atoms joined by a chain of `sep` bonds through dummy atoms so they are a pair."""
    n = sep + 1
    lig = _Lig()
    tn = sorted(set(names) | {"C"}, key=list(TYPE_TABLE).index)
    lig.type_names = tn
    types = [tn.index("C")] * n
    types[0] = tn.index(names[0]); types[-1] = tn.index(names[1])
    lig.types = np.array(types, np.int32)
    ch = np.zeros(n, np.float32); ch[0] = q[0]; ch[-1] = q[1]
    lig.charges = ch
    lig.xyz = np.array([[1.5 * i, 0.3 * (i % 2), 0] for i in range(n)], np.float32)
    lig.bonds = np.array([(i, i + 1) for i in range(n - 1)], np.int32)
    rot = np.zeros(n - 1, np.uint8); rot[n // 2 - 1] = 1
    lig.rotatable = rot
    return lig


def prob(lig, tp=None):
    g = constant_grid(4, 1.0, 0.0, type_names=lig.type_names)
    if tp is not None:
        return oracle.Problem(g, lig, type_params=tp)
    return oracle.Problem(g, lig)


def test_lj_minimum_is_minus_eps(orc):
    P = prob(two_atoms(("C", "N")))
    req = 0.5 * (4.0 + 3.5)
    eps = math.sqrt(float(np.float32(0.150)) * float(np.float32(0.160)))
    # zero out desolvation for the check: use a table with S = V = 0
    tp = np.array([[TYPE_TABLE[t][0], TYPE_TABLE[t][1], 0.0, 0.0] for t in P.grid.type_names], np.float32)
    roles = np.array([TYPE_TABLE[t][4] for t in P.grid.type_names], np.int32)
    P = prob(two_atoms(("C", "N")), (tp, roles))
    i, j = 0, P.N - 1
    req = 0.5 * (float(np.float32(4.0)) + float(np.float32(3.5)))
    e, dE = P.pair_energy(i, j, req * req)
    assert abs(e + eps) < 1e-12
    assert abs(dE) < 1e-12                                   # stationary at r_eq


def test_hbond_minimum_is_minus_eps(orc):
    lig = two_atoms(("HD", "OA"))
    tp = np.array([[TYPE_TABLE[t][0], TYPE_TABLE[t][1], 0.0, 0.0] for t in lig.type_names], np.float32)
    roles = np.array([TYPE_TABLE[t][4] for t in lig.type_names], np.int32)
    P = prob(lig, (tp, roles))
    req = 0.5 * (float(np.float32(2.0)) + float(np.float32(3.2)))
    eps = math.sqrt(float(np.float32(0.02)) * float(np.float32(0.2)))
    e, dE = P.pair_energy(0, P.N - 1, req * req)
    assert abs(e + eps) < 1e-12                              # 5x^12 - 6x^10 = -1 at x = 1
    assert abs(dE) < 1e-12


def test_electrostatic_example(orc):
    lig = two_atoms(("C", "C"), q=(1.0, 1.0))
    tp = np.zeros((len(lig.type_names), 4), np.float32); tp[:, 0] = 1.0
    roles = np.zeros(len(lig.type_names), np.int32)
    P = prob(lig, (tp, roles))                                # eps = 0, S = V = 0
    e, _ = P.pair_energy(0, P.N - 1, 4.0)
    assert abs(e - 20.753976875) < 1e-12                     # 332.06363 / 16


def test_empty_pair_list(orc):
    lig = make_ligand(6, 0, 7)                               # rigid: no pairs
    P = prob(lig)
    assert P.P == 0
    e, g = P.intra(lig.xyz)
    assert e == 0.0 and not g.any()


def test_rigid_motion_invariance(orc):
    lig = make_ligand(40, 8, 3)
    P = prob(lig)
    rng = np.random.default_rng(0)
    genes = np.concatenate([rng.uniform(-3, 3, 3), rng.uniform(0, 6, 3 + P.T)])
    r = P.pose(genes)
    e0, _ = P.intra(r)
    from scipy.spatial.transform import Rotation
    R = Rotation.from_rotvec(rng.normal(size=3)).as_matrix()
    e1, _ = P.intra(r @ R.T + rng.normal(size=3) * 10)
    assert abs(e1 - e0) <= 1e-9 * max(1.0, abs(e0))


def test_decay_far(orc):
    P = prob(two_atoms(("C", "C")))
    req = 4.0
    tp = np.array([[TYPE_TABLE[t][0], TYPE_TABLE[t][1], 0.0, 0.0] for t in P.grid.type_names], np.float32)
    roles = np.zeros(len(P.grid.type_names), np.int32)
    P = prob(two_atoms(("C", "C")), (tp, roles))
    e, _ = P.pair_energy(0, P.N - 1, (50 * req) ** 2)
    assert abs(e) < 1e-6


def test_clamp(orc):
    P = prob(two_atoms(("C", "N"), q=(0.3, -0.2)))
    e1, d1 = P.pair_energy(0, P.N - 1, 1e-6)
    e2, d2 = P.pair_energy(0, P.N - 1, 5e-5)
    e3, _ = P.pair_energy(0, P.N - 1, 1e-4)
    assert e1 == e2 == e3 and d1 == 0.0 and d2 == 0.0        # constant for r <= 0.01 Å


@pytest.mark.parametrize("names,q", [(("C", "N"), (0.3, -0.2)), (("HD", "NA"), (0.3, -0.4)),
                                     (("OA", "A"), (-0.4, 0.1))])
def test_pair_derivative_central_difference(orc, names, q):
    P = prob(two_atoms(names, q))
    for r in (2.5, 3.3, 4.1, 6.0, 9.0):
        rho2 = r * r; h = 1e-6 * rho2
        _, dE = P.pair_energy(0, P.N - 1, rho2)
        ep, _ = P.pair_energy(0, P.N - 1, rho2 + h)
        em, _ = P.pair_energy(0, P.N - 1, rho2 - h)
        fd = (ep - em) / (2 * h)
        assert abs(dE - fd) <= 1e-6 * max(1.0, abs(fd))
