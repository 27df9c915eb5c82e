"""Pins for the oracle's D4 intermolecular energy ("three-dimensional grid")."""
import numpy as np
import pytest

from gen import constant_grid, multilinear_grid
from gen.synth import Grid
import oracle


class _Lig:
    pass


def one_atom(q=0.0, t=0, type_names=("C",)):
    lig = _Lig()
    lig.type_names = list(type_names); lig.types = np.array([t], np.int32)
    lig.charges = np.array([q], np.float32); lig.xyz = np.zeros((1, 3), np.float32)
    lig.bonds = np.zeros((0, 2), np.int32); lig.rotatable = np.zeros(0, np.uint8)
    return lig


def random_grid(n=6, spacing=0.5, seed=0, nt=1):
    rng = np.random.default_rng(seed)
    maps = rng.uniform(-3, 3, size=(nt + 2, n, n, n)).astype(np.float32)
    return Grid(n=(n, n, n), spacing=spacing, origin=np.array([-1.0, 0.5, 2.0], np.float32),
                type_names=["C", "A", "N"][:nt], maps=maps)


def test_exact_at_nodes(orc):
    g = random_grid()
    P = oracle.Problem(g, one_atom())
    for (i, j, k) in [(0, 0, 0), (5, 5, 5), (2, 3, 4), (5, 0, 3)]:
        r = g.origin.astype(np.float64) + g.spacing * np.array([i, j, k])
        e, _ = P.inter_atom(0, r)
        assert e == float(g.maps[0, k, j, i])          # storage i + nx (j + ny k)


def test_multilinear_exactness(orc):
    # dyadic coefficients: every node value is exact in float32 (maps are float32 data)
    coef = (0.25, -1.125, 0.75, 2.0, 0.0625, -0.375, 0.3125, 0.015625)
    n, s = 7, 0.5
    g = multilinear_grid(n, s, [0.5, -1.0, 0.25], coef)
    P = oracle.Problem(g, one_atom())
    a, b, c, d, e, f, gg, h = coef
    rng = np.random.default_rng(3)
    for _ in range(200):
        u = rng.uniform(0, n - 1, 3)
        r = g.origin.astype(np.float64) + s * u
        x, y, z = u
        val = a + b * x + c * y + d * z + e * x * y + f * y * z + gg * x * z + h * x * y * z
        grad_u = np.array([b + e * y + gg * z + h * y * z, c + e * x + f * z + h * x * z,
                           d + f * y + gg * x + h * x * y])
        E, G = P.inter_atom(0, r)
        assert abs(E - val) < 1e-9 * max(1, abs(val))
        assert np.abs(G - grad_u / s).max() < 1e-9 * max(1, np.abs(grad_u).max() / s)


def test_cell_centre_mean(orc):
    maps = np.zeros((3, 2, 2, 2), np.float32)
    maps[0] = np.arange(8, dtype=np.float32).reshape(2, 2, 2)     # corners 0..7
    g = Grid(n=(2, 2, 2), spacing=1.0, origin=np.zeros(3, np.float32), type_names=["C"], maps=maps)
    P = oracle.Problem(g, one_atom())
    assert P.inter_atom(0, [0.5, 0.5, 0.5])[0] == 3.5


def test_convex_bound(orc):
    g = random_grid(seed=5)
    P = oracle.Problem(g, one_atom())
    rng = np.random.default_rng(7)
    for _ in range(200):
        u = rng.uniform(0, 5, 3)
        i = np.minimum(np.floor(u).astype(int), 4)
        corners = g.maps[0, i[2]:i[2] + 2, i[1]:i[1] + 2, i[0]:i[0] + 2]
        e, _ = P.inter_atom(0, g.origin + g.spacing * u)
        assert corners.min() - 1e-9 <= e <= corners.max() + 1e-9


def test_spec_single_atom_examples(orc):
    maps = np.zeros((3, 3, 3, 3), np.float32)
    maps[0, 1, 1, 1] = -1.25; maps[1, 1, 1, 1] = 2.0; maps[2, 1, 1, 1] = 0.5
    g = Grid(n=(3, 3, 3), spacing=1.0, origin=np.zeros(3, np.float32), type_names=["C"], maps=maps)
    P0 = oracle.Problem(g, one_atom(q=0.0))
    assert P0.inter_atom(0, [1, 1, 1])[0] == -1.25                  # S:187 (desolv x |q| = 0)
    P1 = oracle.Problem(g, one_atom(q=1.0))
    assert P1.inter_atom(0, [1, 1, 1])[0] == 1.25                   # -1.25 + 2.0 + 0.5
    Pm = oracle.Problem(g, one_atom(q=-1.0))
    assert Pm.inter_atom(0, [1, 1, 1])[0] == -1.25 - 2.0 + 0.5      # |q| on the desolvation map


def test_out_of_grid_penalty(orc):
    g = constant_grid(5, 1.0, 0.0)
    P = oracle.Problem(g, one_atom())
    hi = g.origin + 4.0
    e, G = P.inter_atom(0, hi + np.array([10.0, 0.0, 0.0]) - np.array([0, 2, 2]))
    assert e == 1e5 * (1 + 10.0)
    assert np.allclose(G, [1e5, 0, 0])
    r = g.origin + np.array([-3.0, -4.0, 2.0])                      # corner region, d = 5
    e, G = P.inter_atom(0, r)
    assert abs(e - 1e5 * 6.0) < 1e-6
    assert np.allclose(G, 1e5 * np.array([-0.6, -0.8, 0.0]))


def test_upper_face_is_inside(orc):
    g = random_grid(seed=9)
    P = oracle.Problem(g, one_atom())
    r = g.origin.astype(np.float64) + g.spacing * np.array([5.0, 2.0, 5.0])   # u = n-1 on x and z
    e, _ = P.inter_atom(0, r)
    assert e == float(g.maps[0, 5, 2, 5])


def test_identity_pose_on_nodes(orc):
    """E_inter at the identity pose with atoms on nodes = sum of direct node lookups (NS)."""
    g = random_grid(n=8, spacing=1.0, seed=2, nt=3)
    lig = _Lig()
    lig.type_names = ["C", "A", "N"]
    nodes = np.array([[1, 2, 3], [2, 2, 3], [3, 2, 3], [3, 3, 3], [4, 3, 5]])
    lig.types = np.array([0, 1, 2, 1, 0], np.int32)
    lig.charges = np.array([0.3, -0.2, 0.1, -0.4, 0.2], np.float32)
    lig.xyz = (g.origin + nodes * g.spacing).astype(np.float32)
    lig.bonds = np.array([(0, 1), (1, 2), (2, 3), (3, 4)], np.int32)
    lig.rotatable = np.array([0, 1, 0, 0], np.uint8)
    P = oracle.Problem(g, lig)
    genes = np.zeros(P.G); genes[:3] = lig.xyz.astype(np.float64).mean(axis=0)
    r = P.pose(genes)
    E, _ = P.inter(r)
    direct = 0.0
    for a, (i, j, k) in enumerate(nodes):
        q = float(lig.charges[a])
        direct += g.maps[lig.types[a], k, j, i] + q * g.maps[3, k, j, i] + abs(q) * g.maps[4, k, j, i]
    assert abs(E - direct) < 1e-9
