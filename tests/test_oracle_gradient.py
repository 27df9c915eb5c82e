"""Pins for the oracle's D7 genotype gradient (NS "analytic gradient back-projected to
genotype space"): central differences of the oracle's energy, which is itself pinned
by test_oracle_inter/intra; plus closed-form special cases."""
import math

import numpy as np
import pytest

from gen import config_inputs, make_ligand, multilinear_grid, random_genotypes
from gen.synth import Grid, retype
import oracle


def fd_grad(P, x, h=1e-6):
    g = np.zeros_like(x)
    for j in range(x.shape[0]):
        xp = x.copy(); xp[j] += h
        xm = x.copy(); xm[j] -= h
        g[j] = (P.energy(xp, grad=False)["E"] - P.energy(xm, grad=False)["E"]) / (2 * h)
    return g


def test_gradient_vs_central_differences_tiny(orc):
    cfg, lig, grid = config_inputs("tiny")
    P = oracle.Problem(grid, lig)
    X = random_genotypes(grid, P.T, 80, seed=11, frac_out=0.1, shrink=0.3).astype(np.float64)
    checked = 0
    for x in X:
        res = P.energy(x)
        fm, cm = P.margins(res["xyz"])
        if fm < 1e-3 or cm < 1e-3:
            continue                      # boundary pose: one-sided derivative
        fd = fd_grad(P, x)
        scale = max(np.abs(res["grad"]).max(), 1.0)
        assert np.abs(fd - res["grad"]).max() <= 1e-5 * scale + 1e-9 * abs(res["E"]) / 1e-6
        checked += 1
    assert checked >= 60


def test_gradient_multilinear_grid_smooth(orc):
    """A globally multilinear map is C-infinity across cell faces: no rejection needed."""
    lig = make_ligand(16, 5, 2)
    coef = (0.25, -0.125, 0.0625, 0.5, 0.015625, -0.03125, 0.0078125, 0.001953125)
    n, s = 40, 0.5
    g = multilinear_grid(n, s, [-10.0, -10.0, -10.0], coef, type_names=lig.type_names)
    g.maps[-2] = g.maps[0] * 0.5; g.maps[-1] = g.maps[0] * 0.25
    P = oracle.Problem(g, lig)
    rng = np.random.default_rng(4)
    for _ in range(10):
        x = np.concatenate([rng.uniform(-2, 2, 3), rng.uniform(-2 * math.pi, 4 * math.pi, 3 + P.T)])
        res = P.energy(x)
        fd = fd_grad(P, x)
        assert np.abs(fd - res["grad"]).max() <= 1e-6 * max(np.abs(res["grad"]).max(), 1.0)


@pytest.mark.parametrize("name", ["1stp", "3ce3"])
def test_gradient_vs_central_differences_configs(orc, name):
    cfg, lig, grid = config_inputs(name)
    P = oracle.Problem(grid, lig)
    X = random_genotypes(grid, P.T, 12, seed=5, frac_out=0.1).astype(np.float64)
    checked = 0
    for x in X:
        res = P.energy(x)
        fm, cm = P.margins(res["xyz"])
        if fm < 1e-3 or cm < 1e-3:
            continue
        fd = fd_grad(P, x)
        scale = max(np.abs(res["grad"]).max(), 1.0)
        assert np.abs(fd - res["grad"]).max() <= 1e-5 * scale + 1e-9 * abs(res["E"]) / 1e-6
        checked += 1
    assert checked >= 6


def test_alpha_zero_kills_axis_gradient(orc):
    cfg, lig, grid = config_inputs("tiny")
    P = oracle.Problem(grid, lig)
    x = random_genotypes(grid, P.T, 1, seed=3, frac_out=0.0)[0].astype(np.float64)
    x[5] = 0.0
    g = P.energy(x)["grad"]
    assert g[3] == 0.0 and g[4] == 0.0


def test_empty_moved_set_zero_torsion_gradient(orc):
    lig = make_ligand(8, 2, 1)
    # make the last bond (to a terminal atom) rotatable as an extra torsion: its moved set is empty
    deg = np.bincount(lig.bonds.reshape(-1), minlength=8)
    k = [e for e, (x, y) in enumerate(lig.bonds) if deg[x] == 1 or deg[y] == 1][0]
    lig.rotatable = lig.rotatable.copy(); lig.rotatable[k] = 1
    cfg, _, grid = config_inputs("tiny")
    lig = retype(lig, grid.type_names)
    P = oracle.Problem(grid, lig)
    empty = [t for t in range(P.T) if not P.topo["moved"][t].any()]
    assert empty
    x = random_genotypes(grid, P.T, 1, seed=8, frac_out=0.0)[0].astype(np.float64)
    g = P.energy(x)["grad"]
    for t in empty:
        assert g[6 + t] == 0.0


def test_energy_at_given_pose(orc):
    """or_energy_at (DESIGN.md §3 reading 22b): at the oracle's own pose it is or_energy
    bit for bit; at any other pose its energy is or_inter + or_intra of that pose (both
    pinned by test_oracle_inter/intra) and its translation gradient is the sum of their
    per-atom gradients (D7: dE/dt = sum_a g_a); the rotational and torsional components
    are invariant under a common translation of pose and t (D7 uses r_a - t, r_a - r_ak)."""
    cfg, lig, grid = config_inputs("1stp")
    P = oracle.Problem(grid, lig)
    X = random_genotypes(grid, P.T, 20, seed=19, frac_out=0.0, shrink=0.3).astype(np.float64)
    rng = np.random.default_rng(3)
    for x in X:
        own = P.energy(x)
        at = P.energy_at(x, own["xyz"])
        assert at["E"] == own["E"] and np.array_equal(at["grad"], own["grad"])
        r = own["xyz"] + rng.normal(0, 0.05, own["xyz"].shape)       # a perturbed pose
        at = P.energy_at(x, r)
        ei, gi = P.inter(r)
        ep, gp = P.intra(r)
        assert abs(at["E"] - (ei + ep)) <= 1e-12 * max(1.0, abs(ei + ep))
        assert np.allclose(at["grad"][:3], (gi + gp).sum(0), rtol=1e-12, atol=1e-9)
        # common shift of the pose and t: rotational/torsional projections only see
        # differences (the energy itself changes: the grid is fixed)
        sh = np.array([0.3, -0.2, 0.1])
        xs = x.copy(); xs[:3] += sh
        a2 = P.energy_at(xs, r + sh)
        g_exp_t = (P.inter(r + sh)[1] + P.intra(r + sh)[1])
        Gam = np.cross(r + sh - xs[:3], g_exp_t).sum(0)
        assert abs(a2["grad"][5] - Gam @ np.array([np.sin(x[4]) * np.cos(x[3]), np.sin(x[4]) * np.sin(x[3]),
                                                   np.cos(x[4])])) <= 1e-9 * max(1.0, np.abs(Gam).max())
