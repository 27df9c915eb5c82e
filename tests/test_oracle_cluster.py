"""Pins for the oracle's NEXT-3 clustering (reading D12: AutoDock's
cluster analysis of the per-run best poses with plain RMSD).

Pinned by: rigid translations (RMSD of a pose translated by d is exactly |d|), a
hand-built case whose clusters follow from the definition, permutation invariance of the
partition, the degenerate cases (one pose, all identical, tolerance 0), and the
energy-order / NaN / tie rules."""
import numpy as np
import pytest

import oracle


def base_pose(N=12, seed=0):
    return np.random.default_rng(seed).normal(0.0, 2.0, (N, 3))


def test_rmsd_of_translation_is_its_length(orc):
    X = base_pose()
    for d in [np.array([0.0, 0.0, 0.0]), np.array([1.0, 2.0, 2.0]), np.array([-0.3, 0.4, 0.0])]:
        assert oracle.rmsd(X, X + d) == pytest.approx(np.linalg.norm(d), abs=1e-12)
    # one atom displaced by s out of N: RMSD = s / sqrt(N)
    Y = X.copy(); Y[3, 1] += 6.0
    assert oracle.rmsd(X, Y) == pytest.approx(6.0 / np.sqrt(12), abs=1e-12)


def test_hand_built_clusters(orc):
    X = base_pose()
    shifts = [0.0, 1.0, 5.0, 1.5, 5.5, 20.0, 2.5]     # along x
    E = [-9.0, -8.0, -7.5, -7.0, -6.0, -5.0, -4.0]
    poses = np.stack([X + np.array([s, 0, 0]) for s in shifts])
    nc, c, r, rank = oracle.cluster(poses, E, 2.0)
    # seeds in energy order: 0 (x=0); 1 joins 0 (1.0); 2 new (5.0 from 0); 3 joins 0 (1.5);
    # 4 joins 2 (0.5); 5 new; 6 is 2.5 from seed 0 and 2.5 from seed 2 -> new
    assert nc == 4
    assert list(c) == [0, 0, 1, 0, 1, 2, 3]
    np.testing.assert_allclose(r, [0.0, 1.0, 0.0, 1.5, 0.5, 0.0, 0.0], atol=1e-12)
    assert list(rank) == list(range(7))


def test_joins_first_cluster_in_creation_order(orc):
    X = base_pose()
    poses = np.stack([X, X + [3.0, 0, 0], X + [1.5, 0, 0]])
    nc, c, r, _ = oracle.cluster(poses, [-3.0, -2.0, -1.0], 2.0)
    # pose 2 is 1.5 from both seeds: the lowest-numbered cluster wins
    assert nc == 2 and list(c) == [0, 1, 0]


def test_partition_invariant_under_input_permutation(orc):
    rng = np.random.default_rng(4)
    X = base_pose(20, 1)
    n = 40
    poses = np.stack([X + rng.normal(0, 1.5, 3) for _ in range(n)])
    E = rng.normal(-5, 2, n)
    nc, c, r, rank = oracle.cluster(poses, E, 2.0)
    perm = rng.permutation(n)
    nc2, c2, r2, rank2 = oracle.cluster(poses[perm], E[perm], 2.0)
    assert nc == nc2
    np.testing.assert_array_equal(c[perm], c2)
    np.testing.assert_allclose(r[perm], r2, atol=0)
    np.testing.assert_array_equal(rank[perm], rank2)
    # every member is within tol of its seed; every seed is >= tol from earlier seeds
    seeds = {}
    for k in np.argsort(rank):
        if c[k] not in seeds:
            for s in seeds.values():
                assert oracle.rmsd(poses[k], poses[s]) >= 2.0
            seeds[c[k]] = k
        assert oracle.rmsd(poses[k], poses[seeds[c[k]]]) < 2.0


def test_degenerate_cases(orc):
    X = base_pose()
    assert oracle.cluster(X[None], [1.0], 2.0)[0] == 1
    same = np.stack([X] * 5)
    nc, c, r, _ = oracle.cluster(same, [0.0] * 5, 2.0)
    assert nc == 1 and (c == 0).all() and (r == 0).all()
    nc, c, _, _ = oracle.cluster(same, [0.0] * 5, 0.0)     # tolerance 0: r < 0 never holds
    assert nc == 5 and list(c) == [0, 1, 2, 3, 4]
    nc, c, _, _ = oracle.cluster(np.zeros((0, 4, 3)), np.zeros(0), 2.0)
    assert nc == 0


def test_energy_order_nan_and_ties(orc):
    X = base_pose()
    poses = np.stack([X + [10.0 * i, 0, 0] for i in range(4)])
    nc, c, r, rank = oracle.cluster(poses, [np.nan, -1.0, -1.0, -2.0], 2.0)
    assert list(rank) == [3, 1, 2, 0]          # -2 first, tie -1/-1 by index, NaN last
    assert list(c) == [3, 1, 2, 0]
