"""Pins for the oracle's D1 topology.

The pair rule and torsion orientation are checked against hand cases and against
an independent Floyd-Warshall / union-find construction written here in numpy.
"""
import numpy as np
import pytest

from gen import make_ligand


def chain(n):
    return np.array([(i, i + 1) for i in range(n - 1)], np.int32)


def test_four_atom_chain_no_pairs(orc):
    t = orc.topology(4, chain(4), np.array([0, 1, 0], np.uint8))
    assert t["T"] == 1
    assert t["pairs"].shape[0] == 0


def test_six_atom_chain_pairs(orc):
    # 0-1-2-3-4-5 with rotatable 2-3 -> pairs {(0,4), (0,5), (1,5)} (SURVEY §8(c) D1 pins)
    t = orc.topology(6, chain(6), np.array([0, 0, 1, 0, 0], np.uint8))
    assert [tuple(p) for p in t["pairs"]] == [(0, 4), (0, 5), (1, 5)]
    # root fragment tie {0,1,2} vs {3,4,5} -> smallest atom index side is root
    assert (t["tor_a"][0], t["tor_b"][0]) == (2, 3)
    assert list(np.nonzero(t["moved"][0])[0]) == [4, 5]


def test_rigid_ligand(orc):
    t = orc.topology(5, chain(5), np.zeros(4, np.uint8))
    assert t["T"] == 0 and t["pairs"].shape[0] == 0


def test_ring_bond_rejected(orc):
    bonds = np.array([(0, 1), (1, 2), (2, 3), (3, 0), (3, 4)], np.int32)
    with pytest.raises(ValueError):
        orc.topology(5, bonds, np.array([1, 0, 0, 0, 0], np.uint8))
    # the exocyclic bond is a bridge and is accepted
    t = orc.topology(5, bonds, np.array([0, 0, 0, 0, 1], np.uint8))
    assert t["T"] == 1 and (t["tor_a"][0], t["tor_b"][0]) == (3, 4)


def test_disconnected_and_bad_index_rejected(orc):
    with pytest.raises(ValueError):
        orc.topology(4, np.array([(0, 1), (2, 3)], np.int32), np.zeros(2, np.uint8))
    with pytest.raises(ValueError):
        orc.topology(3, np.array([(0, 1), (1, 5)], np.int32), np.zeros(2, np.uint8))
    with pytest.raises(ValueError):
        orc.topology(3, np.array([(0, 1), (1, 1)], np.int32), np.zeros(2, np.uint8))


def test_star_nested_moved_sets(orc):
    # big root fragment 0..3 (star), a branch 3-4-5-6 with two rotatable bonds 3-4, 5-6 ... and 4-5 rigid
    bonds = np.array([(0, 1), (0, 2), (0, 3), (3, 4), (4, 5), (5, 6), (6, 7)], np.int32)
    rot = np.array([0, 0, 0, 1, 0, 1, 0], np.uint8)
    t = orc.topology(8, bonds, rot)
    assert t["T"] == 2
    # parent first (depth 1) then child (depth 2)
    assert list(t["depth"]) == [1, 2]
    assert (t["tor_a"][0], t["tor_b"][0]) == (3, 4)
    assert (t["tor_a"][1], t["tor_b"][1]) == (5, 6)
    m0 = set(np.nonzero(t["moved"][0])[0]); m1 = set(np.nonzero(t["moved"][1])[0])
    assert m0 == {5, 6, 7} and m1 == {7}
    assert m1 <= m0


def _independent(n, bonds, rot):
    """Floyd-Warshall distances + union-find fragments, written independently."""
    INF = 10 ** 6
    D = np.full((n, n), INF, np.int64)
    np.fill_diagonal(D, 0)
    for x, y in bonds:
        D[x, y] = D[y, x] = 1
    for k in range(n):
        D = np.minimum(D, D[:, k:k + 1] + D[k:k + 1, :])
    par = list(range(n))

    def find(a):
        while par[a] != a:
            par[a] = par[par[a]]
            a = par[a]
        return a
    for (x, y), r in zip(bonds, rot):
        if not r:
            par[find(x)] = find(y)
    fr = [find(a) for a in range(n)]
    pairs = [(i, j) for i in range(n) for j in range(i + 1, n) if D[i, j] >= 4 and fr[i] != fr[j]]
    return D, fr, pairs


@pytest.mark.parametrize("n,t,seed", [(8, 2, 1), (16, 5, 2), (40, 8, 3), (70, 15, 4), (25, 6, 11), (55, 12, 12)])
def test_pairs_match_floyd_warshall(orc, n, t, seed):
    lig = make_ligand(n, t, seed)
    top = orc.topology(n, lig.bonds, lig.rotatable)
    D, fr, pairs = _independent(n, lig.bonds, lig.rotatable)
    assert [tuple(p) for p in top["pairs"]] == pairs
    assert top["T"] == t
    # moved sets: far side of each bond, nested or disjoint, parents before children
    for k in range(top["T"]):
        a, b = top["tor_a"][k], top["tor_b"][k]
        mk = set(np.nonzero(top["moved"][k])[0])
        assert a not in mk and b not in mk
        # far side: atoms closer to b than to a (tree: bridge splits the graph)
        far = {v for v in range(n) if D[b, v] < D[a, v]}
        assert mk == far - {b}
        for j in range(k + 1, top["T"]):
            mj = set(np.nonzero(top["moved"][j])[0])
            assert mj <= mk or not (mj & mk)
            # child after parent: no later torsion contains an earlier axis in its moved set
            assert a not in mj and b not in mj


def test_c0_pair_count_at_least_four(orc):
    lig = make_ligand(8, 2, 1)
    assert orc.topology(8, lig.bonds, lig.rotatable)["pairs"].shape[0] >= 4
