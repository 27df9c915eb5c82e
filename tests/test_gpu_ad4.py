"""GPU parity of the NEXT-2 scoring variant D5-AD4 (dock_params.scoring = DOCK_SF_AD4;
DESIGN.md §11): the dk::ad4 kernels through the C ABI vs the oracle's or_pair_energy_ad4
on the same seeded inputs.

Tolerances are the NS ones used for D5 (test_gpu_parity.py).  Extra exclusions, counted:
a pose with a pair within 1e-4 Å of a cutoff (8 or 20.48 Å; the energy jumps there) is
excluded from energy and gradient parity; a pair within 1e-4 Å of a smoothing kink
(r_eq +- 0.25 Å; the force jumps there) only from gradient parity.
"""
import numpy as np
import pytest

import oracle
from gen import config_inputs, random_genotypes
from test_gpu_parity import CONFIGS_LS, assert_parity, compare_at_pose, e_tol, near_reference_genotypes

pytestmark = pytest.mark.gpu

_CACHE = {}


@pytest.fixture(scope="module")
def dock():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2203_02096_b200._build import build
    build()
    import paper_2203_02096_b200 as d
    return d


def setup(dock, name, **kw):
    key = (name, tuple(sorted(kw.items())))
    if key not in _CACHE:
        cfg, lig, grid = config_inputs(name)
        d = dock.Docker.from_inputs(grid, lig, scoring=dock.SF_AD4, **kw)
        _CACHE[key] = (cfg, lig, grid, d, oracle.Problem(grid, lig, sf={}))
    return _CACHE[key]


def cut_margin(P, xyz):
    pr = P.topo["pairs"]
    if len(pr) == 0:
        return 1e300
    r = np.linalg.norm(xyz[pr[:, 0]] - xyz[pr[:, 1]], axis=1)
    return float(np.minimum(np.abs(r - 8.0), np.abs(r - 20.48)).min())


@pytest.mark.parametrize("name,n", [("tiny", 2000), ("1stp", 1000), ("3ce3", 400), ("7cpa", 200), ("pm", 300),
                                    ("pl", 100)])
def test_ad4_energy_gradient_pose_parity(dock, name, n):
    cfg, lig, grid, d, P = setup(dock, name)
    X = random_genotypes(grid, d.T, n, seed=2000 + n, frac_out=0.05)
    X[:5, 6:] = 0.0                                    # a few folded (clash) poses
    E, Gd, xyz = d.eval(X, grad=True, xyz=True)
    E0, _, xyz0 = d.eval(X, grad=False, xyz=True)      # energy-only kernel path
    assert np.isfinite(E).all() and np.isfinite(E0).all() and np.isfinite(Gd).all()
    cut = lambda r: cut_margin(P, r) < 1e-4             # noqa: E731  (energy jumps at a cutoff)
    c, fails = compare_at_pose(P, grid, X, E, xyz, Gd=Gd, extra_excl=cut, kink=True)
    assert_parity(c, fails, name + " AD4 energy+gradient")
    c0, fails0 = compare_at_pose(P, grid, X, E0, xyz0, extra_excl=cut)
    assert_parity(c0, fails0, name + " AD4 energy-only")
    ex_e, ex_g = c["ex_e"], c["ex_g"]
    assert ex_e + ex_g < 0.35 * n     # PL: 5,190 pairs x 4 kinks each -> ~1/4 of poses near one


def test_ad4_differs_from_d5(dock):
    """The variant is really in use: D5 and AD4 contexts disagree, each matching its oracle."""
    cfg, lig, grid, d, P = setup(dock, "3ce3")
    d5 = dock.Docker.from_inputs(grid, lig)
    X = near_reference_genotypes(grid, lig, d.T, 32, seed=3)
    Ea, _, _ = d.eval(X)
    E5, _, _ = d5.eval(X)
    P5 = oracle.Problem(grid, lig)
    for i in range(32):
        assert abs(Ea[i] - E5[i]) > 1e-2
        assert abs(E5[i] - P5.energy(X[i].astype(np.float64), grad=False)["E"]) <= e_tol(E5[i])


@pytest.mark.parametrize("name", ["tiny", "3ce3", "7cpa"])
def test_ad4_energy_terms_and_binding_estimate(dock, name):
    cfg, lig, grid, d, P = setup(dock, name)
    X = near_reference_genotypes(grid, lig, d.T, 64, seed=5)
    inter, intra, dG = d.eval_terms(X)
    E, _, _ = d.eval(X)
    for i in range(64):
        ref = P.energy(X[i].astype(np.float64), grad=False)
        assert abs(inter[i] - ref["inter"]) <= e_tol(ref["inter"])
        assert abs(intra[i] - ref["intra"]) <= e_tol(ref["intra"])
        assert abs(dG[i] - P.binding_dG(ref["inter"])) <= e_tol(ref["inter"])
        assert abs(inter[i] + intra[i] - E[i]) <= e_tol(E[i])


@pytest.mark.parametrize("name,iters", [("tiny", 5), ("3ce3", 3), ("7cpa", 2)])
def test_ad4_adadelta_steps(dock, name, iters):
    """AD4 ADADELTA: every iteration of the GPU's trajectory at NS tolerance against the
    oracle's D5-AD4 at the GPU's pose (kinks / cutoffs excluded and counted)."""
    from test_gpu_ls_protocol import ad_trajectory_check
    cfg, lig, grid, d, P = setup(dock, name)
    X = near_reference_genotypes(grid, lig, d.T, 64, seed=31)
    g, E, ev = d.ls_step(0, X, np.full(64, 1e30, np.float32), iters)
    assert (ev == iters).all()
    ad_trajectory_check(d, P, grid, X, iters, f"AD4 {name}", kink=True,
                        extra_excl=lambda r: cut_margin(P, r) < 1e-4)


@pytest.mark.parametrize("name", ["1stp", "pm"])
def test_ad4_solis_wets_steps(dock, name):
    from test_gpu_ls_protocol import sw_free_run_check
    cfg, lig, grid, d, P = setup(dock, name, ls_method=1)
    n = 48
    X = random_genotypes(grid, d.T, n, seed=41, frac_out=0.0, shrink=0.2)
    E0 = np.array([P.energy(x, grad=False)["E"] for x in X], np.float32)
    sw_free_run_check(d, P, grid, X, E0, 20, 9, 2, 4, np.arange(n, dtype=np.int32) * 3, f"AD4 {name}")


@pytest.mark.parametrize("name,runs,budget", [("1stp", 8, 40_000), ("7cpa", 3, 60_000)])
def test_ad4_full_run_sampled_outputs(dock, name, runs, budget):
    """Full-size configs with the AD4 scoring: every run's best energy equals the oracle's
    AD4 energy of the returned genotype, the accounting holds, and the run is
    bit-reproducible."""
    cfg, lig, grid, d, P = setup(dock, name, ls_method=CONFIGS_LS[name][0], ls_rate=CONFIGS_LS[name][1],
                                 ls_max_iters=300)
    r = d.run(cfg.pop, runs, budget, 42)
    r2 = d.run(cfg.pop, runs, budget, 42)
    assert np.array_equal(r["best_E"], r2["best_E"]) and np.array_equal(r["best_genes"], r2["best_genes"])
    assert (r["evals"] >= budget).all()
    for i in range(runs):
        ref = P.energy(r["best_genes"][i].astype(np.float64), grad=False)["E"]
        assert abs(ref - r["best_E"][i]) <= e_tol(ref)
        assert np.isfinite(r["best_E"][i])


def test_ad4_screen_matches_single_runs(dock):
    from gen import hts_ligands
    from gen.synth import TYPE_NAMES, make_grid
    ligs = hts_ligands(5, seed=9)
    grid = make_grid(24, 0.5, list(TYPE_NAMES), seed=77)
    kw = dict(scoring=dock.SF_AD4, ls_method=0, ls_rate=0.25, ls_max_iters=20)
    out = dock.screen(grid, ligs, 24, 2, 3000, 11, devices=[0], slots_per_device=2, **kw)
    assert (out["status"] == 0).all()
    for i in (0, 2, 4):
        di = dock.Docker.from_inputs(grid, ligs[i], **kw)
        r = di.run(24, 2, 3000, 11, ligand_id=i, xyz=False)
        assert out["best_E"][i] == r["best_E"].min()
        di.close()
