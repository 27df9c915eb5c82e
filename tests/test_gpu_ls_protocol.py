"""GPU parity of the local searches by the SURVEY.md §8(c) parity protocol (rows a7, a8).

* Solis-Wets, "fed" mode (dock_sw_trace with fed energies): both sides run D9 on the SAME
  candidate energies (float32 values, so the comparisons agree exactly), so every
  accept/reject decision, every rho and the evaluation count must agree bit-exactly with
  the oracle's or_solis_wets_traced; the genes within FP32 rounding of the double search.
  This runs the production kernels: k_ls_sw (depth 1), the speculative k_ls_sw_tree
  (depth 2, 3) and the cooperative split trees.
* Solis-Wets, free running: the GPU's outcome trace against the oracle's on the real
  energies.  Every divergence must start at a near-tie: at the first differing iteration
  some evaluated candidate has |E_c - E_x| within twice the NS energy tolerance (the two
  sides' energies differ by up to that), or a candidate pose touches the box face (the
  D4.5 penalty jumps there).
* ADADELTA, fed (dock_ad_trace with fed energies and gradients): the D10 update and best
  tracking on identical inputs, every iterate within FP32 rounding of the oracle's.
* ADADELTA, the GPU's own trajectory: every iteration's energy and gradient at NS
  tolerance against the oracle at the GPU's pose of that point.  Free-running divergence
  from the oracle's own trajectory must follow a one-sided-gradient pose (cell face,
  clamp) or a gradient whose NS tolerance already exceeds the gene tolerance.
"""
import math

import numpy as np
import pytest

import oracle
from gen import config_inputs, random_genotypes
from test_gpu_parity import box_margin, e_tol, near_reference_genotypes

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def dock():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2203_02096_b200._build import build
    build()
    import paper_2203_02096_b200 as d
    return d


def fed_table(rng, E0, n, iters, p_accept=0.35, stall_rows=()):
    """Float32 candidate energies for n individuals x iters iterations x 2 candidates:
    a mix of improvements and rejections; rows in stall_rows reject everything (rho
    contracts until rho < rho_min stops the search)."""
    T = np.empty((n, iters, 2), np.float32)
    for i in range(n):
        level = float(E0[i])
        for it in range(iters):
            for c in range(2):
                if i in stall_rows or rng.random() > p_accept:
                    T[i, it, c] = np.float32(level + abs(rng.normal(0, 2.0)) + 1e-3)
                else:
                    T[i, it, c] = np.float32(level - abs(rng.normal(0, 0.5)))
            level = min(level, float(T[i, it].min()))
    return T


def insert_ties(T, E0, pp, slots, G, seed, run, gen, every=5):
    """Exact ties E_c == E_x (D9: strict '<' rejects them) at every `every`-th iteration:
    E_x before an iteration depends on the trajectory, so each tie is placed on the
    oracle's fed trajectory so far (entries before it are unchanged)."""
    n, iters, _ = T.shape
    for i in range(n):
        for it in range(2, iters, every):
            _, _, _, to, _, tE = oracle.solis_wets_traced(None, pp, seed, 0, run, gen, int(slots[i]),
                                                          np.zeros(G), float(E0[i]), bowl=np.zeros(G),
                                                          fed=T[i].astype(np.float64))
            if to[it] < 0:
                break
            T[i, it, (it // every) % 2] = np.float32(tE[it, 0])    # E_x before iteration it
    return T


@pytest.mark.parametrize("name,depth,split", [("tiny", 1, 0), ("1stp", 1, 0), ("1stp", 2, 0), ("1stp", 3, 0),
                                              ("3ce3", 2, 0), ("pm", 2, 2), ("pm", 1, 4)])
def test_sw_fed_decisions_bit_exact(dock, name, depth, split):
    cfg, lig, grid = config_inputs(name)
    d = dock.Docker.from_inputs(grid, lig, ls_method=1, sw_depth=depth, sw_split=split)
    n, iters = 24, 120
    rng = np.random.default_rng(100 + depth)
    X = random_genotypes(grid, d.T, n, seed=7, frac_out=0.0, shrink=0.2)
    E0 = rng.normal(-3, 1, n).astype(np.float32)
    slots = (np.arange(n, dtype=np.int32) * 11 + 3)
    seed, run, gen = 1234, 6, 9
    pp = oracle.params(ls_max_iters=iters)
    T = fed_table(rng, E0, n, iters, stall_rows=(1, 5))
    T = insert_ties(T, E0, pp, slots, d.G, seed, run, gen)
    g, E, ev, to, tr = d.sw_trace(X, E0, iters, seed=seed, run=run, gen=gen, slots=slots, fed=T)
    ties = 0
    for i in range(n):
        x, Eo, evo, oto, otr, otE = oracle.solis_wets_traced(None, pp, seed, 0, run, gen, int(slots[i]), X[i],
                                                             float(E0[i]), bowl=np.zeros(d.G),
                                                             fed=T[i].astype(np.float64))
        assert np.array_equal(to[i], oto), (i, np.nonzero(to[i] != oto)[0][:5])      # every decision
        ex = oto >= 0
        assert np.array_equal(tr[i][ex].astype(np.float64), otr[ex]), i               # rho schedule (exact)
        assert ev[i] == evo and E[i] == np.float32(Eo), (i, ev[i], evo, E[i], Eo)      # count, energy
        assert np.abs(g[i] - x).max() <= 1e-4 * max(1.0, np.abs(x).max()), i           # genes: FP32 rounding
        ties += int(np.sum((otE[:, 1] == otE[:, 0]) | (otE[:, 2] == otE[:, 0])))
    assert (to[1] == -1).any() and (to[5] == -1).any()       # stalled rows stopped at rho < rho_min
    assert ties >= n, ties                                   # exact ties were exercised
    d.close()


def _first_diff(a, b):
    k = np.nonzero(a != b)[0]
    return int(k[0]) if k.size else -1


def sw_free_run_check(d, P, grid, X, E0, iters, seed, run, gen, slots, label):
    """The GPU's Solis-Wets outcome trace (dock_sw_trace, free running) against the oracle's
    (or_solis_wets_traced): identical trajectories agree in evaluations and energy; every
    divergence starts at a near-tie (an evaluated candidate within twice the energy tolerance
    of E_x) or at the box face.  Returns (identical, diverged)."""
    g, E, ev, to, tr = d.sw_trace(X, E0, iters, seed=seed, run=run, gen=gen, slots=slots)
    _, _, gxyz = d.eval(g, grad=False, xyz=True)
    pp = oracle.params(ls_max_iters=iters)
    same = diverged = 0
    unexplained = []
    for i in range(X.shape[0]):
        assert E[i] <= E0[i]                                  # never worsens
        x, Eo, evo, oto, otr, otE = oracle.solis_wets_traced(P, pp, seed, 0, run, gen, int(slots[i]), X[i],
                                                             float(E0[i]))
        k = _first_diff(to[i], oto)
        if k < 0:
            same += 1
            assert ev[i] == evo, (label, i, ev[i], evo)
            # identical decisions: the genes agree within the FP32 rounding of the iterates, and
            # the GPU's final energy is at NS tolerance against the oracle at the GPU's final
            # pose (reading 22b; the oracle's own energy at its own genes differs from that only
            # by its sensitivity to the genes' FP32 drift)
            assert np.abs(g[i] - x).max() <= 1e-4 * max(1.0, np.abs(x).max()), (label, i)
            at = P.energy_at(g[i].astype(np.float64), gxyz[i].astype(np.float64), grad=False)["E"]
            assert abs(E[i] - at) <= e_tol(at), (label, i, E[i], at)
            continue
        diverged += 1
        Ex, E1, E2 = otE[k]
        near = abs(E1 - Ex) <= 2 * e_tol(Ex) or (not math.isnan(E2) and abs(E2 - Ex) <= 2 * e_tol(Ex))
        if not near:
            xo, _, _, _, _, _ = oracle.solis_wets_traced(P, oracle.params(ls_max_iters=k), seed, 0, run, gen,
                                                        int(slots[i]), X[i], float(E0[i]))
            near = box_margin(grid, P.pose(xo)) < 5e-3 or E1 > 5e4 or (not math.isnan(E2) and E2 > 5e4)
        if not near:
            unexplained.append((i, k, Ex, E1, E2, int(to[i][k]), int(oto[k])))
    print(f"SW free run {label}: {same} identical, {diverged} diverged, unexplained {unexplained}")
    assert not unexplained, unexplained
    return same, diverged


def ad_trajectory_check(d, P, grid, X, K, label, kink=False, extra_excl=None):
    """Every iteration of the GPU's own ADADELTA trajectory (dock_ad_trace) at NS tolerance
    against the oracle at the GPU's pose of that point (energy and gradient)."""
    from test_gpu_parity import assert_parity, compare_at_pose
    n = X.shape[0]
    g, E, ev, tx, tE, tg = d.ad_trace(X, np.full(n, 1e30, np.float32), K)
    assert (ev == K).all()                                    # exactly max_iters evaluations (D10)
    flat = tx.reshape(-1, d.G)
    _, _, xyz = d.eval(flat, grad=False, xyz=True)
    c, fails = compare_at_pose(P, grid, flat, tE.reshape(-1), xyz, Gd=tg.reshape(-1, d.G), kink=kink,
                               extra_excl=extra_excl)
    assert_parity(c, fails, f"{label} ADADELTA trajectory ({n} x {K} iterations)")
    # best tracking: the returned energy is the minimum of the traced ones (lowest iteration on ties)
    assert np.array_equal(E, tE.min(axis=1))
    return c


@pytest.mark.parametrize("name,depth", [("1stp", 0), ("1stp", 1), ("3ce3", 0), ("pm", 0)])
def test_sw_free_run_divergence_only_at_near_ties(dock, name, depth):
    cfg, lig, grid = config_inputs(name)
    d = dock.Docker.from_inputs(grid, lig, ls_method=1, sw_depth=depth)
    P = oracle.Problem(grid, lig)
    n, iters = 48, 80
    X = random_genotypes(grid, d.T, n, seed=41, frac_out=0.0, shrink=0.2)
    E0 = np.array([P.energy(x, grad=False)["E"] for x in X], np.float32)
    same, _ = sw_free_run_check(d, P, grid, X, E0, iters, 9, 2, 4, np.arange(n, dtype=np.int32) * 3,
                                f"{name} depth {depth}")
    assert same >= n // 2, same
    d.close()


@pytest.mark.parametrize("name", ["tiny", "1stp", "7cpa"])
def test_adadelta_fed_update_matches_oracle(dock, name):
    """D10 state machine on identical inputs: (energy, gradient) of every iteration fed to
    k_ls_adadelta (TRACE instantiation) and to or_adadelta_traced.  The best-tracking
    choice and the evaluation count are exact; every iterate within FP32 rounding of the
    double update (3 operations per gene per step, 12 steps)."""
    cfg, lig, grid = config_inputs(name)
    d = dock.Docker.from_inputs(grid, lig)
    n, iters = 32, 12
    rng = np.random.default_rng(17)
    X = random_genotypes(grid, d.T, n, seed=3, frac_out=0.0, shrink=0.2)
    fed = np.empty((n, iters, d.G + 1), np.float32)
    fed[:, :, 0] = rng.normal(0, 3, (n, iters))
    fed[:, :, 1:] = rng.normal(0, 1, (n, iters, d.G)) * 10.0 ** rng.uniform(-4, 2, (n, iters, d.G))
    fed[3, 5, 0] = fed[3, 2, 0]                        # exact tie in best tracking: first stays
    E0 = np.full(n, 1e30, np.float32)
    g, E, ev, tx, tE, tg = d.ad_trace(X, E0, iters, fed=fed)
    pp = oracle.params()
    for i in range(n):
        x, Eo, evo, otx, otE, otg = oracle.adadelta_traced(None, pp, iters, X[i], 1e30, bowl=np.zeros(d.G),
                                                           fed=fed[i].astype(np.float64))
        assert ev[i] == evo == iters
        assert np.array_equal(tE[i], fed[i, :, 0]) and np.array_equal(tg[i], fed[i, :, 1:])
        assert E[i] == np.float32(Eo)                      # best energy: one of the fed values
        assert int(np.argmin(tE[i])) == int(np.argmin(otE))
        scale = np.maximum(1.0, np.abs(otx))
        assert (np.abs(tx[i] - otx) <= 2e-6 * scale * np.arange(1, iters + 1)[:, None]).all(), i
        assert np.abs(g[i] - x).max() <= 2e-6 * iters * max(1.0, np.abs(x).max())
    d.close()


@pytest.mark.parametrize("name,K", [("tiny", 8), ("3ce3", 6), ("7cpa", 5), ("pm", 5)])
def test_adadelta_trajectory_parity_and_free_run(dock, name, K):
    """Every iteration of the GPU's own ADADELTA trajectory (dock_ad_trace: the point,
    energy and gradient k_ls_adadelta evaluated) at NS tolerance against the oracle at the
    GPU's pose of that point; with the fed-update test this pins each step of row a7.  The
    free-running trajectories themselves are chaotic (SURVEY §8(c) unpinned (i)): each
    divergence from the oracle's own trajectory must follow a one-sided-gradient pose (cell
    face / clamp within 1e-4) or a gradient large enough that the NS gradient tolerance
    (1e-3 max|grad|) alone exceeds the gene tolerance of the comparison."""
    cfg, lig, grid = config_inputs(name)
    d = dock.Docker.from_inputs(grid, lig)
    P = oracle.Problem(grid, lig)
    n = 48
    X = near_reference_genotypes(grid, lig, d.T, n, seed=31)
    E0 = np.full(n, 1e30, np.float32)
    g, E, ev, tx, tE, tg = d.ad_trace(X, E0, K)
    flat_x = tx.reshape(-1, d.G)
    _, _, xyz = d.eval(flat_x, grad=False, xyz=True)
    from test_gpu_parity import assert_parity, compare_at_pose
    c, fails = compare_at_pose(P, grid, flat_x, tE.reshape(-1), xyz, Gd=tg.reshape(-1, d.G))
    assert_parity(c, fails, f"{name} ADADELTA trajectory ({n} x {K} iterations)")
    pp = oracle.params()
    same = 0
    why = {"cell face / clamp": 0, "gradient scale": 0, "near-tie": 0}
    unexplained = []
    for i in range(n):
        _, _, _, otx, otE, otg = oracle.adadelta_traced(P, pp, K, X[i], 1e30)
        dev = [np.abs(tx[i, j] - otx[j]).max() / max(1.0, np.abs(otx[j]).max()) for j in range(K)]
        k = next((j for j in range(K) if dev[j] > 1e-3), -1)
        if k < 0:
            same += 1
            continue
        reason = None
        for j in range(k):
            fm, cm = P.margins(P.pose(otx[j]))
            gm = max(1.0, np.abs(otg[j]).max())
            if fm < 1e-4 or cm < 1e-4:
                reason = "cell face / clamp"
            elif 1e-3 * gm > 1e-3 * max(1.0, np.abs(otx[j + 1]).max()):
                reason = "gradient scale"
            elif j > 0 and abs(otE[j] - otE[:j].min()) <= 2 * e_tol(otE[j]):
                reason = "near-tie"
            if reason:
                break
        if reason:
            why[reason] += 1
        else:
            unexplained.append((i, k, [float(v) for v in dev[:k + 1]]))
    print(f"ADADELTA free run {name}: {same}/{n} identical through {K} iterations; divergences: {why}")
    assert not unexplained, unexplained[:3]
    d.close()
