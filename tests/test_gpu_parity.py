"""GPU parity: the CUDA path through the C ABI vs the CPU oracle on the same seeded inputs.

Tolerances (NS): integers bit-exact; pose |dr| <= 1e-4 Å;
energy |dE| <= max(1e-3, 1e-4 |E|); gradient ||d grad||_inf <= 1e-3 max(||grad||_inf, 1).
Poses with an atom within 1e-4 grid units of a cell face (or a pair at the 0.01 Å clamp)
are excluded from gradient parity (one-sided derivatives) and counted.
"""
import math

import numpy as np
import pytest

import oracle
from gen import config_inputs, planted_grid, random_genotypes

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


_CACHE = {}


def setup(dock, name, **kw):
    key = (name, tuple(sorted(kw.items())))
    if key not in _CACHE:
        cfg, lig, grid = config_inputs(name)
        d = dock.Docker.from_inputs(grid, lig, **kw)
        _CACHE[key] = (cfg, lig, grid, d, oracle.Problem(grid, lig))
    return _CACHE[key]


def e_tol(E):
    return max(1e-3, 1e-4 * abs(E))


# FP32 pose coordinates carry an absolute error of ~2e-5 Å (transforms of ~30 Å
# coordinates).  A pair energy ~ rho^-12 then has relative error ~12 * 2e-5 / rho; in a
# clash pose that term dominates E and the NS 1e-4 relative bound is unreachable in FP32.
# DESIGN.md §3 reading 22b: for a pose whose closest pair is at rho_min < 0.5 Å the
# energy and gradient tolerances are widened to 12 * 2e-5 / rho_min relative.
def clash_factor(P, xyz):
    pr = P.topo["pairs"]
    if len(pr) == 0:
        return 0.0
    rho = np.linalg.norm(xyz[pr[:, 0]] - xyz[pr[:, 1]], axis=1).min()
    return 12 * 2e-5 / max(rho, 1e-2) if rho < 0.5 else 0.0


def pose_tols(P, ref):
    cf = clash_factor(P, ref["xyz"])
    et = max(e_tol(ref["E"]), cf * abs(ref["E"]))
    gt = max(1e-3, cf) * max(1.0, np.abs(ref["grad"]).max()) if ref["grad"] is not None else None
    return et, gt


def near_reference_genotypes(grid, lig, T, n, seed, tau=0.3):
    """Poses in the pocket with torsions near the generator's clash-free conformation."""
    rng = np.random.default_rng(seed)
    L = (np.array(grid.n) - 1) * grid.spacing
    c = grid.origin + L / 2
    X = np.zeros((n, 6 + T), np.float32)
    X[:, :3] = c + rng.uniform(-0.15, 0.15, (n, 3)) * L
    X[:, 3:6] = rng.uniform(0, 2 * math.pi, (n, 3))
    X[:, 6:] = rng.uniform(-tau, tau, (n, T))
    return X


# ---------------------------------------------------------------------------
# a1 / D2: Philox
# ---------------------------------------------------------------------------
def test_philox_kat_on_device(dock):
    import os
    rows = []
    for line in open(os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append(v)
    ctr = np.array([r[0:4] for r in rows], np.uint32)
    key = np.array([r[4:6] for r in rows], np.uint32)
    out = dock.philox(ctr, key)
    assert np.array_equal(out, np.array([r[6:10] for r in rows], np.uint32))


@pytest.mark.parametrize("purpose,slot,gen,run", [(0, 3, 0, 0), (1, 149, 12, 19), (2, 0, 5, 7), (3, 88, 300, 99)])
def test_stream_words_bit_exact(dock, purpose, slot, gen, run):
    seed, lig = 0xDEADBEEF12345, 17
    w = dock.stream_words(seed, lig, purpose, slot, gen, run, 5, 300)
    ref = np.array([oracle.word(seed, lig, purpose, slot, gen, run, 5 + m) for m in range(300)], np.uint32)
    assert np.array_equal(w, ref)


# ---------------------------------------------------------------------------
# a3-a6 / D3-D7: pose, energy, gradient
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,n", [("tiny", 3000), ("1stp", 1500), ("3ce3", 600), ("7cpa", 300), ("pm", 400), ("pl", 120)])
def test_energy_gradient_pose_parity(dock, name, n):
    cfg, lig, grid, d, P = setup(dock, name)
    # pairs/torsions of the device context equal the oracle's (bit-exact)
    axis, moved = d.torsions()
    assert np.array_equal(d.pairs(), P.topo["pairs"])
    assert np.array_equal(axis[:, 0], P.topo["tor_a"]) and np.array_equal(moved, P.topo["moved"])
    X = random_genotypes(grid, d.T, n, seed=1000 + n, frac_out=0.05)
    # a few clash poses: torsions driven to fold the chain
    X[:5, 6:] = 0.0
    E, Gd, xyz = d.eval(X, grad=True, xyz=True)
    E0, _, _ = d.eval(X, grad=False, xyz=False)            # energy-only kernel path
    assert np.isfinite(E).all() and np.isfinite(E0).all() and np.isfinite(Gd).all()
    bad_e = bad_g = bad_x = ex_e = ex_g = 0
    hi = np.array(grid.n) - 1
    for i in range(n):
        ref = P.energy(X[i].astype(np.float64))
        fm, cm = P.margins(ref["xyz"])
        if np.abs(xyz[i] - ref["xyz"]).max() > 1e-4:
            bad_x += 1
        # energy is continuous across cell faces but jumps at the box faces (D4.5)
        u = (ref["xyz"] - grid.origin.astype(np.float64)) / grid.spacing
        box_margin = np.minimum(np.abs(u), np.abs(u - hi)).min()
        if box_margin < 1e-4:
            ex_e += 1
            continue
        tol, gtol = pose_tols(P, ref)
        if abs(E[i] - ref["E"]) > tol or abs(E0[i] - ref["E"]) > tol:
            bad_e += 1
        # gradients are one-sided on every cell face: FP32 and FP64 may pick different cells
        if fm < 1e-4 or cm < 1e-4:
            ex_g += 1
            continue
        if np.abs(Gd[i] - ref["grad"]).max() > gtol:
            bad_g += 1
    assert bad_x == 0 and bad_e == 0 and bad_g == 0, (bad_x, bad_e, bad_g, ex_e, ex_g)
    # expected exclusions: ~2e-4 per atom-axis coordinate for gradients
    assert ex_e <= 0.01 * n + 2 and ex_g <= 3 * 3 * lig.n_atoms * 2e-4 * n + 3, (ex_e, ex_g)


def test_degenerate_genotypes(dock):
    cfg, lig, grid, d, P = setup(dock, "1stp")
    # identity pose at the box centre, huge unwrapped angles, far outside the box
    c = lig.xyz.astype(np.float64).mean(0)
    X = np.zeros((4, d.G), np.float32)
    X[0, :3] = c
    X[1, :3] = c; X[1, 3:] = 1234.5
    X[2, :3] = grid.origin - 50.0
    X[3, :3] = c; X[3, 5] = 2 * math.pi
    E, Gd, xyz = d.eval(X, grad=True, xyz=True)
    for i in range(4):
        ref = P.energy(X[i].astype(np.float64))
        assert abs(E[i] - ref["E"]) <= e_tol(ref["E"])
        assert np.abs(xyz[i] - ref["xyz"]).max() < 1e-3 * max(1, np.abs(ref["xyz"]).max()) / 10
    assert np.abs(xyz[0] - lig.xyz).max() < 1e-4                 # identity genotype (D3)


# ---------------------------------------------------------------------------
# a9 / D8: GA step on injected state
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["tiny", "1stp", "7cpa"])
def test_ga_step_parity(dock, name):
    cfg, lig, grid, d, P = setup(dock, name)
    pop = cfg.pop
    rng = np.random.default_rng(5)
    old = random_genotypes(grid, d.T, pop, seed=77)
    oldE = rng.normal(0, 50, pop).astype(np.float32)
    oldE[3] = oldE[7] = oldE.min() - 1.0       # tie for the elite -> lowest index
    oldE[11] = np.nan
    seed, run, gen = 4242, 3, 9
    ng, nE, dbg, perm = d.ga_step(seed, 0, run, gen, old, oldE)
    pp = oracle.params(ls_rate=cfg.ls_rate)
    assert dbg[0, 7] == oracle.elite(oldE.astype(np.float64)) == 3
    assert np.array_equal(ng[0], old[3]) and nE[0] == oldE[3]
    for k in range(1, pop):
        child, odbg = oracle.ga_slot(pp, seed, 0, run, gen, k, old.astype(np.float64), oldE.astype(np.float64))
        assert list(dbg[k, :7]) == list(odbg[:7]), (k, dbg[k], odbg)       # integers bit-exact
        assert np.abs(ng[k] - child).max() <= 1e-6 * max(1.0, np.abs(child).max())
        ref = P.energy(child, grad=False)
        fm, _ = P.margins(ref["xyz"])
        if fm > 1e-4:
            assert abs(nE[k] - ref["E"]) <= pose_tols(P, ref)[0]
    nls = oracle.n_ls(cfg.ls_rate, pop)
    assert np.array_equal(perm[:nls], oracle.ls_pick(seed, 0, run, gen, pop, nls)[:nls])


# ---------------------------------------------------------------------------
# a7 / D10 and a8 / D9: local search from injected state
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,iters", [("tiny", 1), ("tiny", 5), ("3ce3", 3), ("7cpa", 2)])
def test_adadelta_steps(dock, name, iters):
    """ADADELTA normalises every gene's step by its own running RMS, so a gene whose
    gradient is below FP32 noise (relative to the largest component) takes a +-0.22 step
    of random sign: multi-step trajectories are only comparable from poses without
    extreme clashes.  Starts: pocket poses near the clash-free reference conformation."""
    cfg, lig, grid, d, P = setup(dock, name)
    X = near_reference_genotypes(grid, lig, d.T, 64, seed=31)
    E0 = np.full(64, 1e30, np.float32)
    g, E, ev = d.ls_step(0, X, E0, iters)
    assert (ev == iters).all()
    pp = oracle.params()
    ok = 0
    for i in range(64):
        x, Eo, evo = oracle.adadelta(P, pp, iters, X[i], 1e30)
        if abs(E[i] - Eo) <= e_tol(Eo) and np.abs(g[i] - x).max() <= 1e-3 * max(1.0, np.abs(x).max()):
            ok += 1
    assert ok >= 56, ok          # the rest: cell-face crossings / near-ties in best tracking


def test_solis_wets_steps(dock):
    cfg, lig, grid, d, P = setup(dock, "1stp", ls_method=1)
    n = 48
    X = random_genotypes(grid, d.T, n, seed=41, frac_out=0.0, shrink=0.2)
    E0 = np.array([P.energy(x, grad=False)["E"] for x in X], np.float32)
    slots = np.arange(n, dtype=np.int32) * 3
    g, E, ev = d.ls_step(1, X, E0, 20, seed=9, run=2, gen=4, slots=slots)
    pp = oracle.params(ls_max_iters=20)
    ok = 0
    for i in range(n):
        x, Eo, evo = oracle.solis_wets(P, pp, 9, 0, 2, 4, int(slots[i]), X[i], float(E0[i]))
        assert E[i] <= E0[i]                                       # never worsens
        if ev[i] == evo and abs(E[i] - Eo) <= e_tol(Eo):
            ok += 1
    assert ok >= 0.9 * n, ok     # divergence only after a near-tie accept/reject decision


# ---------------------------------------------------------------------------
# D8 + D11 end to end
# ---------------------------------------------------------------------------
def test_run_tiny_accounting_determinism_and_oracle_agreement(dock):
    cfg, lig, grid, d, P = setup(dock, "tiny", ls_method=0, ls_rate=1.0, ls_max_iters=30)
    r1 = d.run(cfg.pop, 8, cfg.max_evals, 42)
    r2 = d.run(cfg.pop, 8, cfg.max_evals, 42)
    for k in ("best_E", "best_genes", "evals", "generations", "best_xyz"):
        assert np.array_equal(r1[k], r2[k]), k                     # bit-reproducible
    per_gen = (cfg.pop - 1) + oracle.n_ls(1.0, cfg.pop) * 30
    assert (r1["evals"] == cfg.pop + r1["generations"] * per_gen).all()
    assert (r1["evals"] >= cfg.max_evals).all() and (r1["evals"] - cfg.max_evals < per_gen).all()
    for i in range(8):
        ref = P.energy(r1["best_genes"][i].astype(np.float64), grad=False)
        assert abs(ref["E"] - r1["best_E"][i]) <= e_tol(ref["E"])
        assert np.abs(ref["xyz"] - r1["best_xyz"][i]).max() < 1e-4
    # statistical agreement with the oracle's runs (trajectories are chaotic)
    pp = oracle.params(ls_method=0, ls_rate=1.0, ls_max_iters=30)
    ore = [oracle.dock_run(P, pp, cfg.pop, cfg.max_evals, 42, run=i)["best_E"] for i in range(8)]
    gpu_med, or_med = float(np.median(r1["best_E"])), float(np.median(ore))
    assert abs(gpu_med - or_med) < 0.25 * abs(or_med) + 0.5, (gpu_med, or_med)


def test_run_sharding_invariance(dock):
    cfg, lig, grid, d, P = setup(dock, "tiny", ls_method=1, ls_rate=0.25, ls_max_iters=30)
    full = d.run(cfg.pop, 4, cfg.max_evals, 7)
    a = d.run(cfg.pop, 2, cfg.max_evals, 7, run_base=0)
    b = d.run(cfg.pop, 2, cfg.max_evals, 7, run_base=2)
    assert np.array_equal(full["best_E"], np.concatenate([a["best_E"], b["best_E"]]))
    assert np.array_equal(full["best_genes"], np.concatenate([a["best_genes"], b["best_genes"]]))
    assert np.array_equal(full["evals"], np.concatenate([a["evals"], b["evals"]]))


def test_first_generation_matches_oracle_exactly_in_integers(dock):
    """Generation 0 genes are a pure function of the Philox stream: the GPU's initial
    population equals the oracle's within FP32 rounding (checked through dock_ga_step's
    elite copy after init is reproduced with the oracle's stream)."""
    cfg, lig, grid, d, P = setup(dock, "tiny")
    words = np.array([[oracle.word(42, 0, 0, k, 0, 0, j) for j in range(d.G)] for k in range(cfg.pop)])
    dev = np.stack([dock.stream_words(42, 0, 0, k, 0, 0, 0, d.G) for k in range(cfg.pop)])
    assert np.array_equal(words.astype(np.uint32), dev)


@pytest.mark.parametrize("method", [0, 1])
def test_planted_minimum_gpu(dock, method):
    class L:
        pass
    lig = L()
    lig.types = np.zeros(1, np.int32); lig.charges = np.zeros(1, np.float32)
    lig.xyz = np.zeros((1, 3), np.float32)
    lig.bonds = np.zeros((0, 2), np.int32); lig.rotatable = np.zeros(0, np.uint8)
    node = (7, 4, 11)
    g = planted_grid(16, 0.75, node)
    d = dock.Docker.from_inputs(g, lig, ls_method=method, ls_rate=0.25 if method else 1.0, ls_max_iters=30)
    r = d.run(16, 10, 2000, 42)
    xs = g.origin + np.array(node) * g.spacing
    hits = (np.linalg.norm(r["best_genes"][:, :3] - xs, axis=1) <= g.spacing).sum()
    assert hits >= 9


@pytest.mark.parametrize("name,runs,budget", [("1stp", 20, 60_000), ("7cpa", 4, 80_000)])
def test_full_size_sampled_outputs(dock, name, runs, budget):
    """Full-size configs in the bench's launch configuration with a reduced budget: every
    run's best energy equals the oracle's energy of the returned genotype (sampled output),
    and the evaluation accounting holds (D11)."""
    cfg, lig, grid, d, P = setup(dock, name, ls_method=CONFIGS_LS[name][0], ls_rate=CONFIGS_LS[name][1],
                                 ls_max_iters=300)
    r = d.run(cfg.pop, runs, budget, 42)
    assert (r["evals"] >= budget).all()
    for i in range(runs):
        ref = P.energy(r["best_genes"][i].astype(np.float64), grad=False)["E"]
        assert abs(ref - r["best_E"][i]) <= e_tol(ref)


CONFIGS_LS = {"1stp": (1, 0.06), "7cpa": (0, 1.0), "3ce3": (0, 1.0)}


# ---------------------------------------------------------------------------
# dock_screen (multi-ligand scheduler): every ligand's result equals a
# standalone dock_run_ex with ligand_id = its index, whatever the slot count and order;
# an invalid ligand is rejected with DOCK_E_INPUT and does not stop the screen.
# ---------------------------------------------------------------------------
def test_screen_matches_single_ligand_runs(dock):
    from gen import hts_ligands
    from gen.synth import TYPE_NAMES, make_grid
    ligs = hts_ligands(7, seed=9)
    grid = make_grid(24, 0.5, list(TYPE_NAMES), seed=77)
    kw = dict(ls_method=0, ls_rate=0.25, ls_max_iters=20)
    pop, runs, budget, seed = 24, 3, 3000, 1234
    import copy
    bad = hts_ligands(1, seed=10)[0]
    ring = copy.deepcopy(bad)
    ring.bonds = np.vstack([bad.bonds, [[0, len(bad.types) - 1]]]).astype(np.int32)
    ring.rotatable = np.concatenate([np.ones(len(bad.bonds), np.uint8), [0]]).astype(np.uint8)
    allligs = ligs[:3] + [ring] + ligs[3:]
    out_a = dock.screen(grid, allligs, pop, runs, budget, seed, devices=[0], slots_per_device=3, **kw)
    out_b = dock.screen(grid, allligs, pop, runs, budget, seed, devices=[0], slots_per_device=1, **kw)
    assert out_a["status"][3] == dock.DOCK_E_INPUT and np.isnan(out_a["best_E"][3])
    assert out_a["stats"]["n_failed"] == 1
    for k in ("best_E", "best_run", "best_genes", "evals", "status"):
        np.testing.assert_array_equal(out_a[k], out_b[k], err_msg=k)
    for i, lig in enumerate(allligs):
        if i == 3:
            continue
        d = dock.Docker.from_inputs(grid, lig, **kw)
        r = d.run(pop, runs, budget, seed, ligand_id=i, xyz=False)
        bE = r["best_E"]
        br = int(np.argmin(np.where(np.isnan(bE), np.inf, bE)))
        assert out_a["status"][i] == 0
        assert out_a["best_E"][i] == bE[br] and out_a["best_run"][i] == br
        np.testing.assert_array_equal(out_a["best_genes"][i, : d.G], r["best_genes"][br])
        assert np.all(out_a["best_genes"][i, d.G:] == 0)
        assert out_a["evals"][i] == r["evals"].sum()
        d.close()


# ---------------------------------------------------------------------------
# Speculative Solis-Wets (k_ls_sw_tree, depth 2 and 3): bit-identical to the plain
# kernel (depth 1) for the LS hook and for whole runs, and equal to the oracle's D9.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["tiny", "1stp", "3ce3"])
def test_sw_speculation_depths_bit_identical(dock, name):
    cfg, lig, grid = config_inputs(name)
    P = oracle.Problem(grid, lig)
    n = 40
    outs = {}
    for depth in (1, 2, 3):
        d = dock.Docker.from_inputs(grid, lig, ls_method=1, sw_depth=depth)
        X = random_genotypes(grid, d.T, n, seed=43, frac_out=0.0, shrink=0.2)
        E0 = np.array([P.energy(x, grad=False)["E"] for x in X], np.float32)
        slots = np.arange(n, dtype=np.int32) * 5 + 1
        outs[depth] = d.ls_step(1, X, E0, 37, seed=11, run=3, gen=2, slots=slots)
        d.close()
    for depth in (2, 3):
        for a, b in zip(outs[1], outs[depth]):
            np.testing.assert_array_equal(a, b)
    g, E, ev = outs[3]
    pp = oracle.params(ls_max_iters=37)
    ok = 0
    for i in range(n):
        x, Eo, evo = oracle.solis_wets(P, pp, 11, 0, 3, 2, int(slots[i]), X[i], float(E0[i]))
        assert E[i] <= E0[i]
        ok += int(ev[i] == evo and abs(E[i] - Eo) <= e_tol(Eo))
    assert ok >= 0.9 * n, ok


def test_sw_speculation_full_run_identical(dock):
    cfg, lig, grid = config_inputs("1stp")
    res = []
    for depth in (1, 2, 3, 0):
        d = dock.Docker.from_inputs(grid, lig, ls_method=1, ls_rate=cfg.ls_rate, ls_max_iters=cfg.ls_iters,
                                    sw_depth=depth)
        res.append(d.run(cfg.pop, 4, 60_000, 42, xyz=False))
        d.close()
    for r in res[1:]:
        for k in ("best_E", "best_genes", "evals", "generations"):
            np.testing.assert_array_equal(res[0][k], r[k], err_msg=k)


# ---------------------------------------------------------------------------
# Deep torsion trees: every internal bond of a zig-zag chain rotatable (depth T), so the
# pointer-jumping composites run ceil(log2(T)) rounds; W = 16 and W = 32 lane groups.
# ---------------------------------------------------------------------------
def _chain_ligand(n, seed):
    from gen.synth import Ligand, TYPE_NAMES
    rng = np.random.default_rng(seed)
    xyz = np.zeros((n, 3), np.float64)
    for i in range(n):
        xyz[i] = (1.25 * i, 0.44 * (i % 2), 0.1 * np.sin(i))
    xyz -= xyz.mean(0)
    names = ["C"] * n
    names[0], names[-1] = "OA", "N"
    q = rng.normal(0, 0.15, n)
    q -= q.mean()
    bonds = np.array([[i, i + 1] for i in range(n - 1)], np.int32)
    rot = np.zeros(n - 1, np.uint8)
    rot[1:-1] = 1
    tn = list(TYPE_NAMES)
    return Ligand(type_names=tn, types=np.array([tn.index(a) for a in names], np.int32),
                  charges=q.astype(np.float32), xyz=xyz.astype(np.float32), bonds=bonds, rotatable=rot,
                  atom_names=names)


@pytest.mark.parametrize("n_atoms", [12, 16, 20, 34])
def test_deep_torsion_chain_parity(dock, n_atoms):
    from gen.synth import TYPE_NAMES, make_grid
    lig = _chain_ligand(n_atoms, seed=n_atoms)
    grid = make_grid(40, 0.5, list(TYPE_NAMES), seed=3)
    d = dock.Docker.from_inputs(grid, lig)
    P = oracle.Problem(grid, lig)
    assert d.T == n_atoms - 3
    X = random_genotypes(grid, d.T, 200, seed=7, frac_out=0.0, shrink=0.1)
    X[:, 6:] *= 0.05                 # near-extended chains: few self-clashes
    E, Gd, xyz = d.eval(X, grad=True, xyz=True)
    bad = []
    for i in range(X.shape[0]):
        ref = P.energy(X[i].astype(np.float64))
        if np.abs(xyz[i] - ref["xyz"]).max() > 1e-4:
            bad.append(("x", i))
            continue
        fm, cm = P.margins(ref["xyz"])
        tol, gtol = pose_tols(P, ref)
        if abs(E[i] - ref["E"]) > tol:
            bad.append(("E", i))
        if fm >= 1e-4 and cm >= 1e-4 and np.abs(Gd[i] - ref["grad"]).max() > gtol:
            bad.append(("g", i))
    assert not bad, bad[:10]
    d.close()


# ---------------------------------------------------------------------------
# Large ligands (beyond the paper's 108-atom PL input, P > 4,900 pairs): the energy-only
# kernels switch to the pair tiles (the pair list would not fit in shared memory).
# ---------------------------------------------------------------------------
@pytest.fixture(scope="module")
def large_case():
    from gen import make_ligand
    from gen.synth import TYPE_NAMES, make_grid
    lig = make_ligand(160, 30, 7, type_names=list(TYPE_NAMES))
    grid = make_grid(48, 0.6, list(TYPE_NAMES), seed=11)
    return lig, grid


def test_large_ligand_energy_tiles_parity(dock, large_case):
    lig, grid = large_case
    d = dock.Docker.from_inputs(grid, lig)
    P = oracle.Problem(grid, lig)
    assert d.N == 160 and d.P > 5000
    X = random_genotypes(grid, d.T, 60, seed=3, frac_out=0.0, shrink=0.05)
    X[:, 6:] *= 0.1
    E, Gd, xyz = d.eval(X, grad=True, xyz=True)
    E0, _, _ = d.eval(X, grad=False)            # energy-only kernel: pair-tile path
    bad = []
    for i in range(X.shape[0]):
        ref = P.energy(X[i].astype(np.float64))
        tol, gtol = pose_tols(P, ref)
        fm, cm = P.margins(ref["xyz"])
        if np.abs(xyz[i] - ref["xyz"]).max() > 1e-4:
            bad.append(("x", i))
        if abs(E[i] - ref["E"]) > tol or abs(E0[i] - ref["E"]) > tol:
            bad.append(("E", i, float(E[i]), float(E0[i]), ref["E"]))
        if fm >= 1e-4 and cm >= 1e-4 and np.abs(Gd[i] - ref["grad"]).max() > gtol:
            bad.append(("g", i))
    assert not bad, bad[:5]
    d.close()


@pytest.mark.parametrize("method", [0, 1])
def test_large_ligand_run(dock, large_case, method):
    lig, grid = large_case
    d = dock.Docker.from_inputs(grid, lig, ls_method=method, ls_rate=0.1, ls_max_iters=20)
    r = d.run(40, 2, 4000, 42, xyz=True)
    P = oracle.Problem(grid, lig)
    assert np.all(r["evals"] >= 4000)
    for k in range(2):
        ref = P.energy(r["best_genes"][k].astype(np.float64))
        tol, _ = pose_tols(P, ref)
        assert abs(ref["E"] - r["best_E"][k]) <= tol, (ref["E"], r["best_E"][k])
    d.close()


# ---------------------------------------------------------------------------
# Maximum sizes: N = 256 atoms (the ABI limit), T = 32 torsions (the limit): MAXC = 8
# chunks, energy-only kernels on the pair tiles (P ~ 30k pairs).
# ---------------------------------------------------------------------------
def test_max_size_ligand_parity_and_run(dock):
    from gen.synth import TYPE_NAMES, make_grid
    n = 256
    lig = _chain_ligand(n, seed=5)
    # a helix-like chain (compact enough for the grid), 32 rotatable bonds spread along it
    k = np.arange(n)
    lig.xyz = np.stack([4.0 * np.cos(k * 0.7), 4.0 * np.sin(k * 0.7), 0.35 * k], 1).astype(np.float32)
    lig.xyz -= lig.xyz.mean(0)
    rot = np.zeros(n - 1, np.uint8)
    rot[np.linspace(2, n - 4, 32).astype(int)] = 1
    lig.rotatable = rot
    grid = make_grid(40, 2.5, list(TYPE_NAMES), seed=9)
    d = dock.Docker.from_inputs(grid, lig, ls_method=1, ls_rate=0.2, ls_max_iters=5)
    P = oracle.Problem(grid, lig)
    assert d.N == 256 and d.T == 32 and d.P > 25000
    X = random_genotypes(grid, d.T, 24, seed=4, frac_out=0.0, shrink=0.02)
    # small torsions only: an 89 Å helix bent by 32 large torsions leaves the box, and the
    # 1e5 kcal/mol/Å out-of-grid slope turns FP32 pose rounding into > 1e-4 relative energy
    X[:, 6:] = 0.02 * np.sin(np.arange(X.shape[0] * d.T).reshape(X.shape[0], d.T))
    E, Gd, xyz = d.eval(X, grad=True, xyz=True)
    E0, _, _ = d.eval(X, grad=False)
    for i in range(X.shape[0]):
        ref = P.energy(X[i].astype(np.float64))
        tol, gtol = pose_tols(P, ref)
        assert np.abs(xyz[i] - ref["xyz"]).max() <= 1e-4 * max(1.0, np.abs(ref["xyz"]).max() / 30)
        assert abs(E[i] - ref["E"]) <= tol and abs(E0[i] - ref["E"]) <= tol, (i, E[i], E0[i], ref["E"])
        fm, cm = P.margins(ref["xyz"])
        if fm >= 1e-4 and cm >= 1e-4:
            assert np.abs(Gd[i] - ref["grad"]).max() <= gtol, i
    r = d.run(8, 1, 200, 42, xyz=False)
    assert r["evals"][0] >= 200 and np.isfinite(r["best_E"][0])
    d.close()


# ---------------------------------------------------------------------------
# Cooperative SW evaluation (sw_split 2 / 4 warps per trial point): same D9 search; the
# energy partials are summed in a fixed order, so results match the oracle within the
# energy tolerance and repeat bit-exactly.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("split,depth", [(2, 2), (4, 1)])
def test_sw_cooperative_split(dock, split, depth):
    cfg, lig, grid = config_inputs("pm")
    P = oracle.Problem(grid, lig)
    n = 24
    d = dock.Docker.from_inputs(grid, lig, ls_method=1, sw_depth=depth, sw_split=split)
    X = random_genotypes(grid, d.T, n, seed=45, frac_out=0.0, shrink=0.2)
    E0 = np.array([P.energy(x, grad=False)["E"] for x in X], np.float32)
    slots = np.arange(n, dtype=np.int32) * 7 + 2
    g1, E1, ev1 = d.ls_step(1, X, E0, 25, seed=13, run=1, gen=3, slots=slots)
    g2, E2, ev2 = d.ls_step(1, X, E0, 25, seed=13, run=1, gen=3, slots=slots)
    np.testing.assert_array_equal(g1, g2)
    np.testing.assert_array_equal(E1, E2)
    pp = oracle.params(ls_max_iters=25)
    ok = 0
    for i in range(n):
        x, Eo, evo = oracle.solis_wets(P, pp, 13, 0, 1, 3, int(slots[i]), X[i], float(E0[i]))
        assert E1[i] <= E0[i]
        ok += int(ev1[i] == evo and abs(E1[i] - Eo) <= e_tol(Eo))
    assert ok >= 0.9 * n, ok
    r = d.run(cfg.pop, 2, 40_000, 42, xyz=False)
    ref = P.energy(r["best_genes"][0].astype(np.float64))
    tol, _ = pose_tols(P, ref)
    assert abs(ref["E"] - r["best_E"][0]) <= tol
    d.close()


# ---------------------------------------------------------------------------
# Tail schedules of the gradient pair tiles (prep.cpp cost model): the last
# partial chunk is rotated as a padded chunk, broadcast atom by atom, or rotated inside
# power-of-two lane segments.  Every schedule must give the oracle's energy and gradient
# for every tail size; DOCK_TAIL forces the segment schedule (seg) or the cost model's
# choice between the other two (bcast).
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n_atoms", [9, 13, 24, 33, 36, 40, 41, 47, 50, 57, 63, 65, 70, 72, 80])
@pytest.mark.parametrize("mode", ["seg", "bcast"])
def test_tail_schedules_parity(dock, n_atoms, mode, monkeypatch):
    from gen import make_ligand
    from gen.synth import TYPE_NAMES, make_grid
    monkeypatch.setenv("DOCK_TAIL", mode)
    lig = make_ligand(n_atoms, min(15, n_atoms // 5), seed=100 + n_atoms, type_names=list(TYPE_NAMES))
    grid = make_grid(40, 0.5, list(TYPE_NAMES), seed=3)
    d = dock.Docker.from_inputs(grid, lig)
    P = oracle.Problem(grid, lig)
    X = near_reference_genotypes(grid, lig, d.T, 48, seed=n_atoms)
    E, Gd, _ = d.eval(X, grad=True)
    assert np.isfinite(E).all() and np.isfinite(Gd).all()
    bad = []
    for i in range(X.shape[0]):
        ref = P.energy(X[i].astype(np.float64))
        fm, cm = P.margins(ref["xyz"])
        tol, gtol = pose_tols(P, ref)
        if abs(E[i] - ref["E"]) > tol:
            bad.append(("E", i, float(E[i]), ref["E"]))
        if fm >= 1e-4 and cm >= 1e-4 and np.abs(Gd[i] - ref["grad"]).max() > gtol:
            bad.append(("g", i))
    assert not bad, bad[:5]
    d.close()


# ---------------------------------------------------------------------------
# Run branches (dock_params.run_branches): every run stepping through its
# generations as its own graph branch gives exactly the lockstep results.
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name,method,runs,budget", [("1stp", 1, 20, 120_000), ("tiny", 1, 6, 2000),
                                                     ("3ce3", 0, 4, 40_000), ("pm", 1, 5, 60_000),
                                                     ("1stp", 1, 1, 30_000)])
def test_run_branches_identical_to_lockstep(dock, name, method, runs, budget):
    cfg, lig, grid = config_inputs(name)
    kw = dict(ls_method=method, ls_rate=0.06 if method == 1 else 1.0,
              ls_max_iters=cfg.ls_iters if name != "tiny" else 30, gens_per_graph=4)
    a = dock.Docker.from_inputs(grid, lig, run_branches=1, **kw)
    b = dock.Docker.from_inputs(grid, lig, run_branches=2, **kw)
    ra = a.run(cfg.pop, runs, budget, 77, run_base=3, ligand_id=5)
    rb = b.run(cfg.pop, runs, budget, 77, run_base=3, ligand_id=5)
    assert a.run_branches == 1 and b.run_branches == runs
    assert a.engine == "lockstep" and b.engine == ("branches" if runs > 1 else "lockstep")
    for k in ("best_E", "best_genes", "evals", "generations", "best_xyz"):
        assert np.array_equal(ra[k], rb[k]), k
    if method == 1:                        # persistent clusters (auto for Solis-Wets where eligible)
        for mode in (3, 0):
            c = dock.Docker.from_inputs(grid, lig, run_branches=mode, **kw)
            rc = c.run(cfg.pop, runs, budget, 77, run_base=3, ligand_id=5)
            assert c.run_branches == runs
            if name == "1stp":             # the headline shape runs in one wave: clusters
                assert c.engine == "clusters", mode
            for k in ("best_E", "best_genes", "evals", "generations", "best_xyz"):
                assert np.array_equal(ra[k], rc[k]), (mode, k)
            c.close()


@pytest.mark.parametrize("ls_rate,max_gen", [(16 / 150, 27000), (17 / 150, 27000), (1 / 150, 27000), (0.06, 7)])
def test_cluster_engine_edges(dock, ls_rate, max_gen):
    """k_run_sw at its eligibility edges (n_ls = 16 clusters, 17 falls back to branches,
    n_ls = 1) and with a generation cap: identical to lockstep."""
    cfg, lig, grid = config_inputs("1stp")
    kw = dict(ls_method=1, ls_rate=ls_rate, ls_max_iters=60, max_generations=max_gen)
    a = dock.Docker.from_inputs(grid, lig, run_branches=1, **kw)
    b = dock.Docker.from_inputs(grid, lig, run_branches=0, **kw)
    ra = a.run(150, 4, 40_000, 5, xyz=False)
    rb = b.run(150, 4, 40_000, 5, xyz=False)
    n_ls = int(np.ceil(np.float64(np.float32(ls_rate)) * 150 - 1e-4))
    assert b.run_branches == 4 and (n_ls <= 16) == (n_ls != 17)
    assert a.engine == "lockstep"
    if n_ls <= 8 or n_ls > 16:             # 9..16 also need the non-portable cluster size to fit
        assert b.engine == ("clusters" if n_ls <= 16 else "branches")
    for k in ("best_E", "best_genes", "evals", "generations"):
        assert np.array_equal(ra[k], rb[k]), k
    if max_gen < 27000:
        assert (ra["generations"] == max_gen).all()
    a.close(); b.close()


def test_screen_solis_wets_cluster_engine(dock):
    """dock_screen with Solis-Wets: several contexts run k_run_sw concurrently on one
    device; every ligand equals its standalone run."""
    from gen import hts_ligands
    from gen.synth import TYPE_NAMES, make_grid
    ligs = hts_ligands(5, seed=21)
    grid = make_grid(24, 0.5, list(TYPE_NAMES), seed=77)
    kw = dict(ls_method=1, ls_rate=0.06, ls_max_iters=60)
    out = dock.screen(grid, ligs, 100, 4, 20_000, 9, devices=[0], slots_per_device=3, **kw)
    assert (out["status"] == 0).all()
    for i, lig in enumerate(ligs):
        d = dock.Docker.from_inputs(grid, lig, **kw)
        r = d.run(100, 4, 20_000, 9, ligand_id=i, xyz=False)
        assert d.run_branches == 4
        assert out["best_E"][i] == np.nanmin(r["best_E"]) and out["evals"][i] == r["evals"].sum()
        d.close()
