"""Pins for the oracle's NEXT-2 variant D5-AD4 (AutoDock4.1-calibrated pair energy;
SURVEY.md §8(f) rank 2).

What pins it to something other than itself:
* with every AD4 change switched off it reduces to D5, which test_oracle_intra pins;
* smoothing equals its definition (minimum of the unsmoothed potential over the window),
  evaluated by brute force on the unsmoothed oracle; the plateau is the LJ minimum -eps;
* the cutoffs zero exactly the terms they name, on the right side;
* the dielectric tends to eps0 at large r, is increasing and positive, and the
  electrostatic energy tends to the screened Coulomb limit w 332.06363 q q / (eps0 r);
* desolvation is even and linear in |q| with the partner's volume as the only route;
* each weight scales only its own term (H-bond vs vdW pairs);
* the genotype gradient matches central differences away from the kinks;
* the intramolecular energy is invariant under rigid motions.
"""
import ctypes as C
import math

import numpy as np
import pytest

from gen import config_inputs, constant_grid, random_genotypes
from gen.synth import TYPE_TABLE
import oracle
from test_oracle_intra import two_atoms

ELEC = 332.06363


def exact_d5():
    """D5_AS_AD4 without float32 rounding (sigma exactly 3.6 as in D5)."""
    c = oracle.CScoring()
    for k, v in oracle.D5_AS_AD4.items():
        setattr(c, k, int(v) if k == "diel" else float(v))
    return c


def prob(lig, sf, zero_sv=False, zero_eps=False):
    g = constant_grid(4, 1.0, 0.0, type_names=lig.type_names)
    tp = np.array([[TYPE_TABLE[t][0], 0.0 if zero_eps else TYPE_TABLE[t][1],
                    0.0 if zero_sv else TYPE_TABLE[t][2], 0.0 if zero_sv else TYPE_TABLE[t][3]]
                   for t in lig.type_names], np.float32)
    roles = np.array([TYPE_TABLE[t][4] for t in lig.type_names], np.int32)
    return oracle.Problem(g, lig, type_params=(tp, roles), sf=sf)


def f32(v):
    return float(np.float32(v))


# ---------------------------------------------------------------------------
# reduction to D5
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", ["tiny", "1stp", "3ce3"])
def test_reduces_to_d5(orc, name):
    cfg, lig, grid = config_inputs(name)
    P5 = oracle.Problem(grid, lig)
    Pa = oracle.Problem(grid, lig, sf=exact_d5())
    X = random_genotypes(grid, P5.T, 40, seed=7, frac_out=0.1).astype(np.float64)
    for x in X:
        a, b = P5.energy(x), Pa.energy(x)
        assert abs(a["E"] - b["E"]) <= 1e-9 * max(1.0, abs(a["E"]))
        assert np.abs(a["grad"] - b["grad"]).max() <= 1e-9 * max(1.0, np.abs(a["grad"]).max())


def test_pair_reduces_to_d5_every_role(orc):
    for names in [("C", "N"), ("HD", "OA"), ("OA", "HD"), ("HD", "NA"), ("OA", "OA")]:
        lig = two_atoms(names, q=(0.4, -0.3))
        P5 = prob(lig, None)
        Pa = prob(lig, exact_d5())
        for rho2 in [1e-5, 0.5, 3.0, 9.0, 30.0, 200.0]:
            e5, d5 = P5.pair_energy(0, P5.N - 1, rho2)
            ea, da = Pa.pair_energy(0, Pa.N - 1, rho2)
            assert abs(e5 - ea) <= 1e-9 * max(1.0, abs(e5)), (names, rho2)
            assert abs(d5 - da) <= 1e-9 * max(1.0, abs(d5)), (names, rho2)


# ---------------------------------------------------------------------------
# smoothing
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("names", [("C", "N"), ("HD", "OA")])
def test_smoothing_is_window_minimum(orc, names):
    lig = two_atoms(names)
    base = dict(w_vdw=1.0, w_hb=1.0, smooth=0.0, cut_vdw=0.0, cut_el=0.0)
    P0 = prob(lig, base, zero_sv=True)                  # unsmoothed vdW / H-bond only
    Ps = prob(lig, dict(base, smooth=0.5), zero_sv=True)
    i, j = 0, P0.N - 1
    req = 0.5 * (f32(TYPE_TABLE[names[0]][0]) + f32(TYPE_TABLE[names[1]][0]))
    for r in np.linspace(0.3, 7.0, 97):
        win = np.linspace(r - 0.25, r + 0.25, 2001)
        win = win[win > 0.01]
        if r - 0.25 <= req <= r + 0.25:
            win = np.append(win, req)
        brute = min(P0.pair_energy(i, j, w * w)[0] for w in win)
        es = Ps.pair_energy(i, j, r * r)[0]
        assert abs(es - brute) <= 1e-9 * max(1.0, abs(brute)), (r, es, brute)


def test_smoothing_plateau_is_lj_minimum(orc):
    for names in [("C", "N"), ("HD", "OA")]:
        lig = two_atoms(names)
        P = prob(lig, dict(w_vdw=1.0, w_hb=1.0, cut_vdw=0.0), zero_sv=True)
        eps = math.sqrt(f32(TYPE_TABLE[names[0]][1]) * f32(TYPE_TABLE[names[1]][1]))
        req = 0.5 * (f32(TYPE_TABLE[names[0]][0]) + f32(TYPE_TABLE[names[1]][0]))
        for r in np.linspace(req - 0.249, req + 0.249, 11):
            e, dE = P.pair_energy(0, P.N - 1, r * r)
            assert abs(e + eps) < 1e-12 and dE == 0.0


# ---------------------------------------------------------------------------
# cutoffs
# ---------------------------------------------------------------------------
def test_vdw_cutoff(orc):
    lig = two_atoms(("C", "N"))
    P = prob(lig, {}, zero_sv=True)                     # charges 0, S = V = 0: vdW only
    e_in = P.pair_energy(0, P.N - 1, 7.999 ** 2)[0]
    e_out, d_out = P.pair_energy(0, P.N - 1, 8.001 ** 2)
    assert e_in < 0.0 and e_out == 0.0 and d_out == 0.0


def test_elec_desolv_cutoff(orc):
    lig = two_atoms(("C", "N"), q=(0.5, 0.5))
    P = prob(lig, {}, zero_eps=True)                    # eps 0: elec + desolv only
    e_in = P.pair_energy(0, P.N - 1, 20.47 ** 2)[0]
    e_out, d_out = P.pair_energy(0, P.N - 1, 20.49 ** 2)
    assert e_in > 0.0 and e_out == 0.0 and d_out == 0.0
    # between the two cutoffs the vdW term is gone but elec stays
    Pv = prob(lig, {})
    assert Pv.pair_energy(0, P.N - 1, 10.0 ** 2)[0] == pytest.approx(P.pair_energy(0, P.N - 1, 10.0 ** 2)[0], rel=1e-12)


# ---------------------------------------------------------------------------
# dielectric and electrostatics
# ---------------------------------------------------------------------------
def test_dielectric_limits_and_shape(orc):
    sf = oracle.scoring()
    e_inf, _ = oracle.dielectric(sf, 1e4)
    assert abs(e_inf - f32(78.4)) < 1e-9
    prev = 0.0
    for r in np.linspace(0.0, 60.0, 601):
        e, de = oracle.dielectric(sf, r)
        assert e > 0.0 and e >= prev and de >= 0.0
        h = 1e-5
        if r > h:
            fd = (oracle.dielectric(sf, r + h)[0] - oracle.dielectric(sf, r - h)[0]) / (2 * h)
            assert abs(fd - de) <= 1e-7 * max(1.0, de)
        prev = e
    # eps(r) = 4r option is the D5 dielectric
    e4, d4 = oracle.dielectric(oracle.scoring(diel=0), 2.5)
    assert e4 == 10.0 and d4 == 4.0


def test_screened_coulomb_limit(orc):
    qi, qj = 0.5, -0.75
    lig = two_atoms(("C", "N"), q=(qi, qj))
    P = prob(lig, dict(cut_el=0.0), zero_sv=True, zero_eps=True)
    w = f32(0.1406)
    for r in [1500.0, 3000.0]:
        e = P.pair_energy(0, P.N - 1, r * r)[0]
        lim = w * ELEC * f32(qi) * f32(qj) / (f32(78.4) * r)
        assert abs(e - lim) <= 1e-9 * abs(lim)
    # antisymmetric in one charge, symmetric in the exchange of the two atoms
    Pm = prob(two_atoms(("C", "N"), q=(-qi, qj)), {}, zero_sv=True, zero_eps=True)
    Px = prob(two_atoms(("N", "C"), q=(qj, qi)), {}, zero_sv=True, zero_eps=True)
    for r in [0.5, 2.0, 7.0]:
        e = P.pair_energy(0, P.N - 1, r * r)[0]
        assert Pm.pair_energy(0, P.N - 1, r * r)[0] == pytest.approx(-e, rel=1e-12)
        assert Px.pair_energy(0, P.N - 1, r * r)[0] == pytest.approx(e, rel=1e-12)


# ---------------------------------------------------------------------------
# charge-dependent desolvation and weights
# ---------------------------------------------------------------------------
def test_desolvation_even_and_linear_in_abs_charge(orc):
    r2 = 3.0 ** 2

    def e_ds(q, names=("OA", "C")):
        # elec removed by w_el = 0; vdW removed by eps = 0
        P = prob(two_atoms(names, q=(q, 0.0)), dict(w_el=0.0), zero_eps=True)
        return P.pair_energy(0, P.N - 1, r2)[0]
    e0, e1, e2, em = e_ds(0.0), e_ds(0.25), e_ds(0.5), e_ds(-0.25)
    assert e1 != e0
    assert abs((e2 - e1) - (e1 - e0)) < 1e-12
    assert abs(e1 - em) < 1e-15
    # the |q_i| term of atom i multiplies V_j: partner with V = 0 -> no charge dependence
    lig = two_atoms(("OA", "C"), q=(0.5, 0.0))
    tp = np.array([[TYPE_TABLE[t][0], 0.0, TYPE_TABLE[t][2], 0.0 if t == "C" else TYPE_TABLE[t][3]]
                   for t in lig.type_names], np.float32)
    roles = np.array([TYPE_TABLE[t][4] for t in lig.type_names], np.int32)
    g = constant_grid(4, 1.0, 0.0, type_names=lig.type_names)
    Pa = oracle.Problem(g, lig, type_params=(tp, roles), sf=dict(w_el=0.0))
    lig0 = two_atoms(("OA", "C"), q=(0.0, 0.0))
    Pb = oracle.Problem(g, lig0, type_params=(tp, roles), sf=dict(w_el=0.0))
    assert Pa.pair_energy(0, Pa.N - 1, r2)[0] == Pb.pair_energy(0, Pb.N - 1, r2)[0]


def test_weights_scale_their_own_term(orc):
    for names, hb in [(("C", "N"), False), (("HD", "OA"), True)]:
        lig = two_atoms(names)
        P1 = prob(lig, {}, zero_sv=True)
        P2 = prob(lig, dict(w_vdw=2 * 0.1662), zero_sv=True)
        P3 = prob(lig, dict(w_hb=2 * 0.1209), zero_sv=True)
        for r in [1.0, 3.0, 6.0]:
            e1 = P1.pair_energy(0, P1.N - 1, r * r)[0]
            e2 = P2.pair_energy(0, P2.N - 1, r * r)[0]
            e3 = P3.pair_energy(0, P3.N - 1, r * r)[0]
            assert e1 != 0.0
            if hb:
                assert e2 == e1 and e3 == pytest.approx(2 * e1, rel=1e-7)
            else:
                assert e3 == e1 and e2 == pytest.approx(2 * e1, rel=1e-7)


# ---------------------------------------------------------------------------
# gradient, invariance, binding estimate
# ---------------------------------------------------------------------------
def fd_grad(P, x, h=1e-6):
    g = np.zeros_like(x)
    for j in range(x.shape[0]):
        xp = x.copy(); xp[j] += h
        xm = x.copy(); xm[j] -= h
        g[j] = (P.energy(xp, grad=False)["E"] - P.energy(xm, grad=False)["E"]) / (2 * h)
    return g


@pytest.mark.parametrize("name", ["tiny", "1stp"])
def test_gradient_vs_central_differences(orc, name):
    cfg, lig, grid = config_inputs(name)
    P = oracle.Problem(grid, lig, sf={})
    X = random_genotypes(grid, P.T, 60, seed=23, frac_out=0.1, shrink=0.3).astype(np.float64)
    checked = 0
    for x in X:
        res = P.energy(x)
        fm, cm = P.margins(res["xyz"])
        if fm < 1e-3 or cm < 1e-3 or P.kink_margin(res["xyz"]) < 1e-3:
            continue
        fd = fd_grad(P, x)
        scale = max(np.abs(res["grad"]).max(), 1.0)
        assert np.abs(fd - res["grad"]).max() <= 1e-5 * scale + 1e-9 * abs(res["E"]) / 1e-6
        checked += 1
    assert checked >= 40


def test_intra_rigid_invariance_and_dG(orc):
    cfg, lig, grid = config_inputs("3ce3")
    P = oracle.Problem(grid, lig, sf={})
    x = random_genotypes(grid, P.T, 1, seed=5)[0].astype(np.float64)
    res = P.energy(x)
    xyz = res["xyz"]
    th = 0.7
    R = np.array([[math.cos(th), -math.sin(th), 0], [math.sin(th), math.cos(th), 0], [0, 0, 1]])
    e0, _ = P.intra(xyz)
    e1, _ = P.intra(xyz @ R.T + np.array([3.0, -2.0, 1.0]))
    assert abs(e0 - e1) <= 1e-9 * max(1.0, abs(e0))
    assert P.binding_dG(res["inter"]) == pytest.approx(res["inter"] + f32(0.2983) * P.T, rel=1e-15)
    assert oracle.Problem(grid, lig).binding_dG(res["inter"]) == res["inter"]
