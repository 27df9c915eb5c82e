"""Pins for the oracle's D3 pose (NS "orientation quaternion")."""
import math

import numpy as np
import pytest
from scipy.spatial.transform import Rotation

from gen import constant_grid, make_ligand
import oracle


def _prob(lig):
    g = constant_grid(8, 1.0, 0.0, type_names=lig.type_names)
    return oracle.Problem(g, lig)


def _chain4():
    class L:  # minimal ligand record
        pass
    lig = L()
    lig.type_names = ["C"]
    lig.types = np.zeros(4, np.int32)
    lig.charges = np.zeros(4, np.float32)
    lig.xyz = np.array([[0, 0, 0], [1.5, 0, 0], [2.0, 1.4, 0], [3.5, 1.4, 0.3]], np.float32)
    lig.bonds = np.array([(0, 1), (1, 2), (2, 3)], np.int32)
    lig.rotatable = np.array([0, 1, 0], np.uint8)
    return lig


def test_identity_genotype(orc):
    lig = make_ligand(16, 5, 2)
    P = _prob(lig)
    c = lig.xyz.astype(np.float64).mean(axis=0)
    genes = np.zeros(P.G); genes[:3] = c
    genes[3] = 0.7; genes[4] = 1.1   # axis irrelevant when alpha = 0
    assert np.abs(P.pose(genes) - lig.xyz.astype(np.float64)).max() < 1e-12


def test_translation_only(orc):
    lig = make_ligand(16, 5, 2)
    P = _prob(lig)
    c = lig.xyz.astype(np.float64).mean(axis=0)
    genes = np.zeros(P.G); genes[:3] = c + np.array([1.0, 2.0, 3.0])
    assert np.abs(P.pose(genes) - (lig.xyz + np.array([1.0, 2.0, 3.0]))).max() < 1e-12


def test_reflection_at_pi(orc):
    lig = _chain4()
    P = _prob(lig)
    X = lig.xyz.astype(np.float64)
    c = X.mean(axis=0)
    genes = np.zeros(P.G); genes[:3] = c; genes[6] = math.pi
    # rotation by pi about the B->C axis: D' = B + (2 u u^T - I)(D - B)
    u = (X[2] - X[1]) / np.linalg.norm(X[2] - X[1])
    Dp = X[1] + (2 * np.outer(u, u) - np.eye(3)) @ (X[3] - X[1])
    out = P.pose(genes)
    assert np.abs(out[3] - Dp).max() < 1e-12
    assert np.abs(out[:3] - X[:3]).max() < 1e-12


def test_x_about_z_quarter_turn(orc):
    class L:
        pass
    lig = L()
    lig.type_names = ["C"]; lig.types = np.zeros(2, np.int32); lig.charges = np.zeros(2, np.float32)
    lig.xyz = np.array([[1, 0, 0], [-1, 0, 0]], np.float32)
    lig.bonds = np.array([(0, 1)], np.int32); lig.rotatable = np.zeros(1, np.uint8)
    P = _prob(lig)
    genes = np.array([0, 0, 0, 0.0, 0.0, math.pi / 2])   # theta = 0 -> n = z
    out = P.pose(genes)
    assert np.abs(out[0] - [0, 1, 0]).max() < 1e-12
    assert np.abs(out[1] - [0, -1, 0]).max() < 1e-12


def test_periodicity_2pi(orc):
    lig = make_ligand(40, 8, 3)
    P = _prob(lig)
    rng = np.random.default_rng(0)
    for _ in range(10):
        g = rng.uniform(-3, 3, P.G)
        g2 = g.copy(); g2[3:] += 2 * math.pi
        assert np.abs(P.pose(g) - P.pose(g2)).max() < 1e-12 * 1e3   # ~1e-9 Å absolute


def _sequential_current_axis(lig, P, genes):
    """SPEC S:117 semantics written independently: torsions applied root -> leaf about the
    CURRENT axis atoms, then the orientation (scipy axis-angle) about the reference
    centroid and the translation."""
    X = lig.xyz.astype(np.float64)
    c = X.mean(axis=0)
    y = X - c
    for k in range(P.T):
        a, b = P.topo["tor_a"][k], P.topo["tor_b"][k]
        A = y[a].copy(); u = y[b] - y[a]; u /= np.linalg.norm(u)
        Rk = Rotation.from_rotvec(genes[6 + k] * u).as_matrix()
        m = P.topo["moved"][k].astype(bool)
        y[m] = A + (y[m] - A) @ Rk.T
    ph, th, al = genes[3:6]
    n = np.array([math.sin(th) * math.cos(ph), math.sin(th) * math.sin(ph), math.cos(th)])
    R = Rotation.from_rotvec(al * n).as_matrix()
    return genes[:3] + y @ R.T


@pytest.mark.parametrize("n,t,seed", [(8, 2, 1), (16, 5, 2), (40, 8, 3), (70, 15, 4)])
def test_reference_axis_equals_current_axis(orc, n, t, seed):
    lig = make_ligand(n, t, seed)
    P = _prob(lig)
    rng = np.random.default_rng(seed)
    for _ in range(5):
        genes = np.concatenate([rng.uniform(-5, 5, 3), rng.uniform(-2 * math.pi, 4 * math.pi, 3 + P.T)])
        assert np.abs(P.pose(genes) - _sequential_current_axis(lig, P, genes)).max() < 1e-10


@pytest.mark.parametrize("n,t,seed", [(40, 8, 3), (70, 15, 4)])
def test_distances_preserved(orc, n, t, seed):
    lig = make_ligand(n, t, seed)
    P = _prob(lig)
    X = lig.xyz.astype(np.float64)
    rng = np.random.default_rng(1)
    genes = np.concatenate([rng.uniform(-5, 5, 3), rng.uniform(-2 * math.pi, 4 * math.pi, 3 + P.T)])
    r = P.pose(genes)
    for x, y in lig.bonds:                                   # bond lengths
        assert abs(np.linalg.norm(r[x] - r[y]) - np.linalg.norm(X[x] - X[y])) < 1e-9
    fr = P.topo["frag"]
    for i in range(n):                                       # intra-fragment distances
        for j in range(i + 1, n):
            if fr[i] == fr[j]:
                assert abs(np.linalg.norm(r[i] - r[j]) - np.linalg.norm(X[i] - X[j])) < 1e-9
