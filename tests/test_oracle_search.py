"""Pins for the oracle's D8-D11 search pieces (P:64 GA + memetic Solis-Wets LS, P:92
sum_evals; NS ADADELTA)."""
import math

import numpy as np
import pytest

from gen import config_inputs, planted_grid
import oracle


def pop_state(pop=40, G=9, seed=0):
    rng = np.random.default_rng(seed)
    return rng.normal(size=(pop, G)), rng.normal(size=pop)


def test_tournament_p1_picks_better_and_ties(orc):
    pp = orc.params(p_tour=1.0, p_cross=0.0, p_mut=0.0)
    genes, E = pop_state()
    genes[:, 0] = np.arange(genes.shape[0])     # identify the parent from gene 0
    for k in range(1, 200):
        child, dbg = orc.ga_slot(pp, 9, 0, 2, 3, k, genes, E)
        A = dbg[0]
        assert child[0] == A
        # recover the two candidates from the words and check A is the better one
        w = [orc.word(9, 0, 1, k, 3, 2, m) for m in range(3)]
        i = orc.below(w[0], 40); j = orc.below(w[1], 39); j += j >= i
        assert A == (i if (E[i] < E[j] or (E[i] == E[j] and i < j)) else j)
    # equal energies -> lower index
    E2 = np.zeros(40)
    for k in range(1, 100):
        _, dbg = orc.ga_slot(pp, 9, 0, 2, 3, k, genes, E2)
        w = [orc.word(9, 0, 1, k, 3, 2, m) for m in range(3)]
        i = orc.below(w[0], 40); j = orc.below(w[1], 39); j += j >= i
        assert dbg[0] == min(i, j)


def test_nan_counts_as_infinity(orc):
    E = np.array([np.nan, 3.0, np.nan, 2.0, 2.0])
    assert orc.elite(E) == 3
    assert orc.elite(np.array([np.nan, np.nan])) == 0


def test_selection_rate_monte_carlo(orc):
    pp = orc.params(p_tour=0.60)
    genes, E = pop_state(pop=150, seed=1)
    better = 0; n = 0
    for k in range(1, 150):
        for gen in range(1, 41):
            _, dbg = orc.ga_slot(pp, 123, 0, 0, gen, k, genes, E)
            for t, A in ((0, dbg[0]), (3, dbg[1])):
                w = [orc.word(123, 0, 1, k, gen, 0, t + m) for m in range(2)]
                i = orc.below(w[0], 150); j = orc.below(w[1], 149); j += j >= i
                b = i if E[i] < E[j] else j
                better += (A == b); n += 1
    assert abs(better / n - 0.60) < 0.01


def test_crossover_exchange_and_cut_points(orc):
    pp = orc.params(p_cross=1.0, p_mut=0.0)
    genes, E = pop_state(seed=2)
    G = genes.shape[1]
    seen_copy = seen_full = False
    for k in range(1, 400):
        child, dbg = orc.ga_slot(pp, 5, 0, 1, 2, k, genes, E)
        A, B, cross, c1, c2 = dbg[:5]
        assert cross == 1 and 0 <= c1 <= c2 <= G
        for j in range(G):                                     # exchange property
            assert child[j] == (genes[B, j] if c1 <= j < c2 else genes[A, j])
        seen_copy |= (c1 == c2)
        seen_full |= (c1 == 0 and c2 == G)
    assert seen_copy                                           # c1 = c2 -> copy of A


def test_mutation_identity_and_rate(orc):
    genes, E = pop_state(pop=150, G=20, seed=3)
    pp0 = orc.params(p_cross=0.0, p_mut=0.0)
    for k in range(1, 50):
        child, dbg = orc.ga_slot(pp0, 5, 0, 1, 2, k, genes, E)
        assert np.array_equal(child, genes[dbg[0]])            # rate 0 -> identity
    pp1 = orc.params(p_cross=0.0, p_mut=1.0, mut_trans=0.0, mut_angle=0.0)
    for k in range(1, 50):
        child, dbg = orc.ga_slot(pp1, 5, 0, 1, 2, k, genes, E)
        assert np.array_equal(child, genes[dbg[0]])            # magnitude 0 -> identity
    pp = orc.params(p_cross=0.0)
    changed = 0; total = 0
    for gen in range(1, 40):
        for k in range(1, 150):
            child, dbg = orc.ga_slot(pp, 77, 0, 0, gen, k, genes, E)
            d = child != genes[dbg[0]]
            changed += d.sum(); total += d.size
            mags = np.abs(child - genes[dbg[0]])
            assert (mags[:3] <= 2.0).all() and (mags[3:] <= np.float32(0.523) + 1e-12).all()
    assert abs(changed / total - 0.02) < 0.002


def test_ls_pick_without_replacement(orc):
    for pop, rate in [(150, 0.06), (16, 0.25), (256, 1.0), (150, 0.1)]:
        nls = orc.n_ls(rate, pop)
        perm = orc.ls_pick(3, 0, 4, 5, pop, nls)
        assert sorted(perm) == list(range(pop))
        assert len(set(perm[:nls])) == nls
    assert orc.n_ls(0.06, 150) == 9 and orc.n_ls(0.1, 150) == 15 and orc.n_ls(1.0, 256) == 256


def test_sum_evals_series(orc):
    assert orc.sum_evals(np.arange(1, 151)) == 11325
    assert orc.sum_evals(np.zeros(10)) == 0


# ---------------------------------------------------------------------------
# D9 Solis-Wets
# ---------------------------------------------------------------------------
def test_sw_bowl_convergence(orc):
    pp = orc.params(ls_max_iters=300)
    ok = 0
    for seed in range(100):
        x0 = np.array([5.0, 0.0, 0.0])                         # distance 5 from the origin
        x, E, ev = orc.solis_wets(None, pp, seed, 0, 0, 1, 0, x0, 25.0, bowl=np.ones(3))
        assert E <= 25.0 and ev <= 600
        ok += E < 0.1 ** 2 * 1.0 or np.linalg.norm(x) < 0.1
    assert ok >= 95


def test_sw_never_worsens_on_docking(orc):
    cfg, lig, grid = config_inputs("tiny")
    P = oracle.Problem(grid, lig)
    pp = orc.params(ls_max_iters=40)
    from gen import random_genotypes
    X = random_genotypes(grid, P.T, 10, seed=4)
    for s, x in enumerate(X):
        E0 = P.energy(x, grad=False)["E"]
        x1, E1, ev = orc.solis_wets(P, pp, 1, 0, 0, 1, s, x, E0)
        assert E1 <= E0 and 1 <= ev <= 80
        assert abs(P.energy(x1, grad=False)["E"] - E1) < 1e-9 * max(1, abs(E1))


# ---------------------------------------------------------------------------
# D10 ADADELTA
# ---------------------------------------------------------------------------
def test_adadelta_first_step_closed_form(orc):
    pp = orc.params()
    rho, eps = float(np.float32(0.8)), float(np.float32(1e-2))
    c = np.array([1.0, 3.0, 0.5])
    x0 = np.array([2.0, -1.0, 0.7])
    g = 2 * c * x0
    x1, E1, ev = orc.adadelta(None, pp, 1, x0, np.inf, bowl=c)
    # best is recorded before the step: best = x0 (E0 < inf); the step itself:
    assert np.array_equal(x1, x0)
    # two iterations: the second evaluation is at x0 + dx
    dx = -np.sqrt(eps) / np.sqrt((1 - rho) * g * g + eps) * g
    x2, E2, ev = orc.adadelta(None, pp, 2, x0, np.sum(c * (x0 + dx) ** 2) + 1e-12, bowl=c)
    assert np.abs(x2 - (x0 + dx)).max() < 1e-15
    assert ev == 2


def test_adadelta_bowl_and_accounting(orc):
    pp = orc.params()
    x, E, ev = orc.adadelta(None, pp, 300, np.array([5.0, 5.0, 5.0]), 75.0, bowl=np.ones(3))
    assert E < 1e-20 and ev == 300
    x, E, ev = orc.adadelta(None, pp, 300, np.array([5.0, 5.0, 5.0]), 75.0 + 5.0 * 0,
                            bowl=np.array([1.0, 10.0, 0.1]))
    assert E <= 261.25 * 1.0 and ev == 300                     # best never worse than input


# ---------------------------------------------------------------------------
# D8 + D11 whole runs
# ---------------------------------------------------------------------------
def test_tiny_run_accounting_and_elitism(orc):
    cfg, lig, grid = config_inputs("tiny")
    P = oracle.Problem(grid, lig)
    for method, rate, iters in [(0, 1.0, 30), (1, 0.25, 30)]:
        pp = orc.params(ls_method=method, ls_rate=rate, ls_max_iters=iters)
        r = orc.dock_run(P, pp, cfg.pop, cfg.max_evals, 42)
        assert r["evals"] >= cfg.max_evals
        if method == 0:
            per_gen = (cfg.pop - 1) + orc.n_ls(rate, cfg.pop) * iters
            assert r["evals"] == cfg.pop + r["generations"] * per_gen
            assert r["evals"] - cfg.max_evals < per_gen         # overshoot <= one generation
        assert abs(P.energy(r["best_genes"], grad=False)["E"] - r["best_E"]) < 1e-9 * max(1, abs(r["best_E"]))
        assert r["best_E"] == r["final_E"].min()


def test_elitism_monotone(orc):
    cfg, lig, grid = config_inputs("tiny")
    P = oracle.Problem(grid, lig)
    pp = orc.params(ls_method=1, ls_rate=0.25, ls_max_iters=20)
    best = []
    for budget in range(200, 1400, 150):
        best.append(orc.dock_run(P, pp, 16, budget, 7)["best_E"])
    # same seed: a longer run extends the shorter one, so the best never gets worse
    assert all(b2 <= b1 for b1, b2 in zip(best, best[1:]))


def test_planted_minimum(orc):
    """a single-atom ligand on a grid with a unique node minimum is found within one
    spacing in >= 9/10 runs."""
    class L:
        pass
    lig = L()
    lig.type_names = ["C"]; lig.types = np.zeros(1, np.int32); lig.charges = np.zeros(1, np.float32)
    lig.xyz = np.zeros((1, 3), np.float32)
    lig.bonds = np.zeros((0, 2), np.int32); lig.rotatable = np.zeros(0, np.uint8)
    node = (7, 4, 11)
    g = planted_grid(16, 0.75, node)
    P = oracle.Problem(g, lig)
    xs = g.origin + np.array(node) * g.spacing
    hits = 0
    for method in (0, 1):
        pp = orc.params(ls_method=method, ls_rate=0.25 if method else 1.0, ls_max_iters=30)
        hits = 0
        for run in range(10):
            r = orc.dock_run(P, pp, 16, 2000, 42, run=run)
            hits += np.linalg.norm(r["best_genes"][:3] - xs) <= g.spacing
        assert hits >= 9
