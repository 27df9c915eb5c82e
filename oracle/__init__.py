"""ctypes wrapper around the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / `--impl reference` leg, never by the product package
(paper_2203_02096_b200), which shares no code with it.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = os.path.join(_HERE, "oracle.c")


def build_oracle(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math: it is the precision reference)."""
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "oracle.h"))):
        tmp = _SO + f".{os.getpid()}.tmp"
        subprocess.check_call(["gcc", "-std=c11", "-O2", "-Wall", "-fPIC", "-shared",
                               "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _SO)
    return _SO


class CScoring(C.Structure):
    _fields_ = [
        ("w_vdw", C.c_double), ("w_hb", C.c_double), ("w_el", C.c_double), ("w_ds", C.c_double),
        ("w_tors", C.c_double), ("qasp", C.c_double), ("smooth", C.c_double),
        ("cut_vdw", C.c_double), ("cut_el", C.c_double), ("diel", C.c_int),
        ("diel_A", C.c_double), ("diel_eps0", C.c_double), ("diel_lambda", C.c_double),
        ("diel_k", C.c_double), ("sigma", C.c_double),
    ]


# NEXT-2: AutoDock 4.1's calibrated free-energy coefficients, charge-dependent
# solvation parameter, smoothing window, cutoffs and Mehler-Solmajer dielectric constants.
AD41 = dict(w_vdw=0.1662, w_hb=0.1209, w_el=0.1406, w_ds=0.1322, w_tors=0.2983, qasp=0.01097,
            smooth=0.5, cut_vdw=8.0, cut_el=20.48, diel=1, diel_A=-8.5525, diel_eps0=78.4,
            diel_lambda=0.003627, diel_k=7.7839, sigma=3.6)
# The same variant with every AD4 change switched off: must reduce to D5.
D5_AS_AD4 = dict(w_vdw=1.0, w_hb=1.0, w_el=1.0, w_ds=1.0, w_tors=0.0, qasp=0.0, smooth=0.0,
                 cut_vdw=0.0, cut_el=0.0, diel=0, diel_A=0.0, diel_eps0=0.0, diel_lambda=0.0,
                 diel_k=0.0, sigma=3.6)


def scoring(**kw):
    """CScoring from AD41 with overrides.  Real values are rounded to float32 (the ABI's
    type), so both sides start from the same numbers."""
    v = dict(AD41); v.update(kw)
    c = CScoring()
    for k, val in v.items():
        setattr(c, k, int(val) if k == "diel" else float(np.float32(val)))
    return c


class CProblem(C.Structure):
    _fields_ = [
        ("nx", C.c_int), ("ny", C.c_int), ("nz", C.c_int),
        ("spacing", C.c_double), ("origin", C.c_double * 3), ("n_types", C.c_int),
        ("maps", C.POINTER(C.c_float)),
        ("tR", C.POINTER(C.c_double)), ("teps", C.POINTER(C.c_double)),
        ("tS", C.POINTER(C.c_double)), ("tV", C.POINTER(C.c_double)),
        ("trole", C.POINTER(C.c_int)),
        ("N", C.c_int), ("type", C.POINTER(C.c_int)), ("q", C.POINTER(C.c_double)),
        ("X", C.POINTER(C.c_double)),
        ("T", C.c_int), ("tor_a", C.POINTER(C.c_int)), ("tor_b", C.POINTER(C.c_int)),
        ("moved", C.POINTER(C.c_ubyte)),
        ("P", C.c_int), ("pairs", C.POINTER(C.c_int)),
        ("sf", C.POINTER(CScoring)),
    ]


class CParams(C.Structure):
    _fields_ = [
        ("p_tour", C.c_double), ("p_cross", C.c_double), ("p_mut", C.c_double),
        ("mut_trans", C.c_double), ("mut_angle", C.c_double),
        ("ls_method", C.c_int), ("ls_rate", C.c_double), ("ls_max_iters", C.c_int),
        ("sw_rho", C.c_double), ("sw_rho_min", C.c_double), ("sw_expand", C.c_double),
        ("sw_contract", C.c_double), ("sw_cons_succ", C.c_int), ("sw_cons_fail", C.c_int),
        ("ad_rho", C.c_double), ("ad_eps", C.c_double), ("max_generations", C.c_int),
    ]


_lib = None


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        L = C.CDLL(_SO)
        P = C.POINTER
        d, i, u32, u64, i64 = C.c_double, C.c_int, C.c_uint32, C.c_uint64, C.c_int64
        L.or_philox4x32_10.argtypes = [P(u32), P(u32), P(u32)]
        L.or_word.argtypes = [u64, u32, u32, u32, u32, u32, u32]
        L.or_word.restype = u32
        L.or_u01.argtypes = [u32]; L.or_u01.restype = d
        L.or_below.argtypes = [u32, u32]; L.or_below.restype = u32
        L.or_topology.argtypes = [i, i, P(i), P(C.c_ubyte), P(i), P(i), P(i), P(C.c_ubyte), P(i),
                                  P(i), P(i), i, P(i)]
        L.or_topology.restype = i
        L.or_topology_verbatim.argtypes = [i, i, P(i), P(i), P(i), i, P(i), P(i), P(i), P(C.c_ubyte), P(i)]
        L.or_topology_verbatim.restype = i
        L.or_pose.argtypes = [P(CProblem), P(d), P(d)]
        L.or_inter_atom.argtypes = [P(CProblem), i, P(d), P(d)]; L.or_inter_atom.restype = d
        L.or_inter.argtypes = [P(CProblem), P(d), P(d)]; L.or_inter.restype = d
        L.or_pair_energy.argtypes = [P(CProblem), i, i, d, P(d)]; L.or_pair_energy.restype = d
        L.or_intra.argtypes = [P(CProblem), P(d), P(d)]; L.or_intra.restype = d
        L.or_pair_energy_ad4.argtypes = [P(CProblem), i, i, d, P(d)]; L.or_pair_energy_ad4.restype = d
        L.or_dielectric.argtypes = [P(CScoring), d, P(d)]; L.or_dielectric.restype = d
        L.or_kink_margin.argtypes = [P(CProblem), P(d)]; L.or_kink_margin.restype = d
        L.or_binding_dG.argtypes = [P(CProblem), d]; L.or_binding_dG.restype = d
        L.or_energy.argtypes = [P(CProblem), P(d), P(d), P(d), P(d)]; L.or_energy.restype = d
        L.or_energy_at.argtypes = [P(CProblem), P(d), P(d), P(d), P(d)]; L.or_energy_at.restype = d
        L.or_margins.argtypes = [P(CProblem), P(d), P(d), P(d)]
        L.or_elite.argtypes = [i, P(d)]; L.or_elite.restype = i
        L.or_ga_slot.argtypes = [P(CParams), u64, u32, u32, u32, u32, i, i, P(d), P(d), P(d), P(i)]
        L.or_n_ls.argtypes = [d, i]; L.or_n_ls.restype = i
        L.or_ls_pick.argtypes = [u64, u32, u32, u32, i, i, P(i)]
        L.or_solis_wets.argtypes = [P(CProblem), P(d), i, P(CParams), u64, u32, u32, u32, u32,
                                    P(d), P(d), P(i64)]
        L.or_adadelta.argtypes = [P(CProblem), P(d), i, P(CParams), i, P(d), P(d), P(i64)]
        L.or_solis_wets_traced.argtypes = [P(CProblem), P(d), i, P(CParams), u64, u32, u32, u32, u32,
                                           P(d), P(d), P(i64), P(d), P(i), P(d), P(d)]
        L.or_adadelta_traced.argtypes = [P(CProblem), P(d), i, P(CParams), i, P(d), P(d), P(i64), P(d), P(d),
                                         P(d), P(d)]
        L.or_init_population.argtypes = [P(CProblem), i, u64, u32, u32, P(d), P(d)]
        L.or_dock_run.argtypes = [P(CProblem), P(CParams), i, i64, u64, u32, u32, P(d), P(d),
                                  P(i64), P(i), P(d)]
        L.or_dock_run.restype = i
        L.or_sum_evals.argtypes = [i, P(i64)]; L.or_sum_evals.restype = i64
        L.or_rmsd.argtypes = [i, P(d), P(d)]; L.or_rmsd.restype = d
        L.or_cluster.argtypes = [i, i, P(d), P(d), d, P(i), P(d), P(i)]; L.or_cluster.restype = i
        _lib = L
    return _lib


def _p(a, ct):
    return a.ctypes.data_as(C.POINTER(ct))


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# D2
# ---------------------------------------------------------------------------
def philox(ctr, key):
    c = np.asarray(ctr, dtype=np.uint32); k = np.asarray(key, dtype=np.uint32)
    out = np.zeros(4, dtype=np.uint32)
    lib().or_philox4x32_10(_p(c, C.c_uint32), _p(k, C.c_uint32), _p(out, C.c_uint32))
    return out


def word(seed, ligand_id, purpose, slot, gen, run, m):
    return int(lib().or_word(seed, ligand_id, purpose, slot, gen, run, m))


def u01(w):
    return float(lib().or_u01(w))


def below(w, n):
    return int(lib().or_below(w, n))


# ---------------------------------------------------------------------------
# D1
# ---------------------------------------------------------------------------
def topology(n_atoms, bonds, rotatable):
    bonds = np.ascontiguousarray(bonds, dtype=np.int32).reshape(-1, 2)
    rot = np.ascontiguousarray(rotatable, dtype=np.uint8)
    T = C.c_int(0); Pn = C.c_int(0)
    ta = np.zeros(32, np.int32); tb = np.zeros(32, np.int32); dep = np.zeros(32, np.int32)
    moved = np.zeros(32 * max(n_atoms, 1), np.uint8)
    cap = max(1, n_atoms * (n_atoms - 1) // 2)
    pairs = np.zeros(2 * cap, np.int32)
    frag = np.zeros(max(n_atoms, 1), np.int32)
    rc = lib().or_topology(n_atoms, bonds.shape[0], _p(bonds, C.c_int), _p(rot, C.c_ubyte),
                           C.byref(T), _p(ta, C.c_int), _p(tb, C.c_int), _p(moved, C.c_ubyte),
                           _p(dep, C.c_int), C.byref(Pn), _p(pairs, C.c_int), cap, _p(frag, C.c_int))
    if rc != 0:
        raise ValueError("oracle topology: invalid ligand")
    t = T.value
    return dict(T=t, tor_a=ta[:t].copy(), tor_b=tb[:t].copy(), depth=dep[:t].copy(),
                moved=moved[: t * n_atoms].reshape(t, n_atoms).copy(),
                pairs=pairs[: 2 * Pn.value].reshape(-1, 2).copy(), frag=frag[:n_atoms].copy())


def topology_verbatim(n_atoms, axis, moved, pairs):
    """D1.7: validate verbatim torsions (axis [T, 2], moved: T index lists) and pairs [P, 2];
    returns the topology dict (as topology(); depth / frag not defined) or raises ValueError."""
    ax = np.ascontiguousarray(axis, dtype=np.int32).reshape(-1)
    T = ax.shape[0] // 2
    off = np.ascontiguousarray(np.concatenate([[0], np.cumsum([len(m) for m in moved])]), dtype=np.int32)
    mv = np.ascontiguousarray(np.concatenate([np.asarray(m, np.int64) for m in moved]) if T else np.zeros(1),
                              dtype=np.int32)
    pr = np.ascontiguousarray(pairs, dtype=np.int32).reshape(-1)
    if pr.size == 0:
        pr = np.zeros(2, np.int32)
    P = np.asarray(pairs).reshape(-1, 2).shape[0]
    ta = np.zeros(max(T, 1), np.int32); tb = np.zeros(max(T, 1), np.int32)
    mo = np.zeros(max(T, 1) * n_atoms, np.uint8); po = np.zeros(max(2 * P, 2), np.int32)
    rc = lib().or_topology_verbatim(n_atoms, T, _p(ax if T else np.zeros(2, np.int32), C.c_int), _p(off, C.c_int),
                                    _p(mv, C.c_int), P, _p(pr, C.c_int), _p(ta, C.c_int), _p(tb, C.c_int),
                                    _p(mo, C.c_ubyte), _p(po, C.c_int))
    if rc != 0:
        raise ValueError("oracle topology_verbatim: invalid torsions / pairs")
    return dict(T=T, tor_a=ta[:T].copy(), tor_b=tb[:T].copy(), moved=mo[: T * n_atoms].reshape(T, n_atoms).copy(),
                pairs=po[: 2 * P].reshape(-1, 2).copy())


# ---------------------------------------------------------------------------
# Problem = grid + type params + ligand (+ D1 topology)
# ---------------------------------------------------------------------------
class Problem:
    """Holds numpy buffers alive and the CProblem view over them."""

    def __init__(self, grid, lig=None, *, types=None, charges=None, xyz=None, bonds=None,
                 rotatable=None, topo=None, type_params=None, sf=None):
        if lig is not None:
            types, charges, xyz, bonds, rotatable = lig.types, lig.charges, lig.xyz, lig.bonds, lig.rotatable
        self.grid = grid
        self.maps = np.ascontiguousarray(grid.maps, dtype=np.float32).reshape(-1)
        if type_params is None:
            tp, roles = grid.type_params()
        else:
            tp, roles = type_params
        tp = np.asarray(tp, dtype=np.float32)
        self.tR = _f64(tp[:, 0]); self.teps = _f64(tp[:, 1])
        self.tS = _f64(tp[:, 2]); self.tV = _f64(tp[:, 3])
        self.trole = np.ascontiguousarray(roles, dtype=np.int32)
        self.type = np.ascontiguousarray(types, dtype=np.int32)
        self.q = _f64(np.asarray(charges, dtype=np.float32))
        self.X = _f64(np.asarray(xyz, dtype=np.float32).reshape(-1))
        N = self.type.shape[0]
        if topo is None:
            topo = topology(N, bonds, rotatable if rotatable is not None else np.zeros(len(bonds), np.uint8))
        self.topo = topo
        self.tor_a = np.ascontiguousarray(topo["tor_a"], dtype=np.int32)
        self.tor_b = np.ascontiguousarray(topo["tor_b"], dtype=np.int32)
        self.moved = np.ascontiguousarray(topo["moved"], dtype=np.uint8).reshape(-1)
        self.pairs = np.ascontiguousarray(topo["pairs"], dtype=np.int32).reshape(-1)
        if self.pairs.size == 0:
            self.pairs = np.zeros(2, np.int32)
        self.N = N; self.T = int(topo["T"]); self.P = int(np.asarray(topo["pairs"]).reshape(-1, 2).shape[0])
        self.G = 6 + self.T
        c = CProblem()
        c.nx, c.ny, c.nz = (int(v) for v in grid.n)
        c.spacing = float(np.float32(grid.spacing))
        for d in range(3):
            c.origin[d] = float(np.float32(grid.origin[d]))
        c.n_types = grid.n_types
        c.maps = _p(self.maps, C.c_float)
        c.tR = _p(self.tR, C.c_double); c.teps = _p(self.teps, C.c_double)
        c.tS = _p(self.tS, C.c_double); c.tV = _p(self.tV, C.c_double)
        c.trole = _p(self.trole, C.c_int)
        c.N = N; c.type = _p(self.type, C.c_int); c.q = _p(self.q, C.c_double); c.X = _p(self.X, C.c_double)
        c.T = self.T; c.tor_a = _p(self.tor_a, C.c_int); c.tor_b = _p(self.tor_b, C.c_int)
        c.moved = _p(self.moved, C.c_ubyte)
        c.P = self.P; c.pairs = _p(self.pairs, C.c_int)
        # sf: None (D5), a CScoring, or a dict of overrides of AD41 (NEXT-2 variant)
        self.sf = scoring(**sf) if isinstance(sf, dict) else sf
        c.sf = C.pointer(self.sf) if self.sf is not None else None
        self.c = c

    def ref(self):
        return C.byref(self.c)

    # D3
    def pose(self, genes):
        g = _f64(genes); out = np.zeros(3 * self.N)
        lib().or_pose(self.ref(), _p(g, C.c_double), _p(out, C.c_double))
        return out.reshape(self.N, 3)

    # D4
    def inter_atom(self, a, r):
        r = _f64(r); g = np.zeros(3)
        e = lib().or_inter_atom(self.ref(), a, _p(r, C.c_double), _p(g, C.c_double))
        return e, g

    def inter(self, xyz):
        x = _f64(xyz).reshape(-1); g = np.zeros_like(x)
        e = lib().or_inter(self.ref(), _p(x, C.c_double), _p(g, C.c_double))
        return e, g.reshape(-1, 3)

    # D5
    def pair_energy(self, i, j, rho2):
        dE = C.c_double(0)
        e = lib().or_pair_energy(self.ref(), i, j, float(rho2), C.byref(dE))
        return e, dE.value

    def intra(self, xyz):
        x = _f64(xyz).reshape(-1); g = np.zeros_like(x)
        e = lib().or_intra(self.ref(), _p(x, C.c_double), _p(g, C.c_double))
        return e, g.reshape(-1, 3)

    # D6 + D7
    def energy(self, genes, grad=True):
        x = _f64(genes); gg = np.zeros(self.G); xyz = np.zeros(3 * self.N); terms = np.zeros(2)
        e = lib().or_energy(self.ref(), _p(x, C.c_double), _p(gg, C.c_double) if grad else None,
                            _p(xyz, C.c_double), _p(terms, C.c_double))
        return dict(E=e, grad=gg if grad else None, xyz=xyz.reshape(self.N, 3), inter=terms[0], intra=terms[1])

    def energy_at(self, genes, xyz, grad=True):
        """D6 + D7 at the given world coordinates xyz [N, 3] (e.g. the GPU's own pose)."""
        x = _f64(genes); r = _f64(xyz).reshape(-1); gg = np.zeros(self.G); terms = np.zeros(2)
        e = lib().or_energy_at(self.ref(), _p(x, C.c_double), _p(r, C.c_double),
                               _p(gg, C.c_double) if grad else None, _p(terms, C.c_double))
        return dict(E=e, grad=gg if grad else None, inter=terms[0], intra=terms[1])

    # NEXT-2
    def kink_margin(self, xyz):
        x = _f64(xyz).reshape(-1)
        return float(lib().or_kink_margin(self.ref(), _p(x, C.c_double)))

    def binding_dG(self, e_inter):
        return float(lib().or_binding_dG(self.ref(), float(e_inter)))

    def margins(self, xyz):
        x = _f64(xyz).reshape(-1); fm = C.c_double(0); cm = C.c_double(0)
        lib().or_margins(self.ref(), _p(x, C.c_double), C.byref(fm), C.byref(cm))
        return fm.value, cm.value


# ---------------------------------------------------------------------------
# D8-D11
# ---------------------------------------------------------------------------
DEFAULTS = dict(p_tour=0.60, p_cross=0.80, p_mut=0.02, mut_trans=2.0, mut_angle=0.523,
                ls_method=0, ls_rate=1.0, ls_max_iters=300, sw_rho=1.0, sw_rho_min=0.01,
                sw_expand=2.0, sw_contract=0.5, sw_cons_succ=4, sw_cons_fail=4,
                ad_rho=0.8, ad_eps=1e-2, max_generations=27000)


def params(**kw):
    """CParams with every real parameter rounded to float32 (the ABI's type), so that
    coin decisions u01(w) < p agree bit-exactly with the FP32 kernels."""
    v = dict(DEFAULTS); v.update(kw)
    p = CParams()
    for k, val in v.items():
        if isinstance(getattr(p, k), float):
            setattr(p, k, float(np.float32(val)))
        else:
            setattr(p, k, int(val))
    return p


def dielectric(sf, r):
    """(eps(r), d eps / dr) of a CScoring (NEXT-2)."""
    de = C.c_double(0)
    e = lib().or_dielectric(C.byref(sf), float(r), C.byref(de))
    return e, de.value


def elite(E):
    E = _f64(E)
    return int(lib().or_elite(E.shape[0], _p(E, C.c_double)))


def ga_slot(pp, seed, ligand_id, run, gen, slot, old_genes, old_E):
    og = _f64(old_genes); oE = _f64(old_E)
    pop, G = og.shape
    child = np.zeros(G); dbg = np.zeros(8, np.int32)
    lib().or_ga_slot(C.byref(pp), seed, ligand_id, run, gen, slot, pop, G, _p(og, C.c_double),
                     _p(oE, C.c_double), _p(child, C.c_double), _p(dbg, C.c_int))
    return child, dbg


def n_ls(ls_rate, pop):
    return int(lib().or_n_ls(float(np.float32(ls_rate)), pop))


def ls_pick(seed, ligand_id, run, gen, pop, nls):
    perm = np.zeros(pop, np.int32)
    lib().or_ls_pick(seed, ligand_id, run, gen, pop, nls, _p(perm, C.c_int))
    return perm


def solis_wets(prob, pp, seed, ligand_id, run, gen, slot, x, E, bowl=None):
    x = _f64(x).copy(); Ec = C.c_double(E); ev = C.c_int64(0)
    G = x.shape[0]
    b = _f64(bowl) if bowl is not None else None
    lib().or_solis_wets(prob.ref() if prob is not None else None,
                        _p(b, C.c_double) if b is not None else None, G, C.byref(pp), seed,
                        ligand_id, run, gen, slot, _p(x, C.c_double), C.byref(Ec), C.byref(ev))
    return x, Ec.value, ev.value


def solis_wets_traced(prob, pp, seed, ligand_id, run, gen, slot, x, E, bowl=None, fed=None):
    """D9 with traces; fed [iters, 2]: the energies of the two candidates of every iteration
    (fed mode), else evaluated.  Returns x, E, evals, outcome [iters] (-1 = not executed),
    rho [iters], Etrace [iters, 3] = (E_x before, E(x+b+d), E(x-b-d) or NaN)."""
    x = _f64(x).copy(); Ec = C.c_double(E); ev = C.c_int64(0)
    G = x.shape[0]; n = pp.ls_max_iters
    b = _f64(bowl) if bowl is not None else None
    ft = _f64(fed).reshape(-1) if fed is not None else None
    to = np.full(max(n, 1), -1, np.int32); tr = np.zeros(max(n, 1)); tE = np.full((max(n, 1), 3), np.nan)
    lib().or_solis_wets_traced(prob.ref() if prob is not None else None,
                               _p(b, C.c_double) if b is not None else None, G, C.byref(pp), seed, ligand_id, run,
                               gen, slot, _p(x, C.c_double), C.byref(Ec), C.byref(ev),
                               _p(ft, C.c_double) if ft is not None else None, _p(to, C.c_int), _p(tr, C.c_double),
                               _p(tE, C.c_double))
    return x, Ec.value, ev.value, to[:n], tr[:n], tE[:n]


def adadelta_traced(prob, pp, iters, x, E, bowl=None, fed=None):
    """D10 with traces; fed [iters, G+1] = (E, grad) per iteration (fed mode) or None.
    Returns x (best), E (best), evals, trace_x [iters, G] (point evaluated at each
    iteration), trace_E [iters], trace_g [iters, G]."""
    x = _f64(x).copy(); Ec = C.c_double(E); ev = C.c_int64(0)
    G = x.shape[0]
    b = _f64(bowl) if bowl is not None else None
    fd = _f64(fed).reshape(-1) if fed is not None else None
    tx = np.zeros((max(iters, 1), G)); tE = np.zeros(max(iters, 1)); tg = np.zeros((max(iters, 1), G))
    lib().or_adadelta_traced(prob.ref() if prob is not None else None,
                             _p(b, C.c_double) if b is not None else None, G, C.byref(pp), iters,
                             _p(x, C.c_double), C.byref(Ec), C.byref(ev),
                             _p(fd, C.c_double) if fd is not None else None, _p(tx, C.c_double),
                             _p(tE, C.c_double), _p(tg, C.c_double))
    return x, Ec.value, ev.value, tx[:iters], tE[:iters], tg[:iters]


def adadelta(prob, pp, iters, x, E, bowl=None):
    x = _f64(x).copy(); Ec = C.c_double(E); ev = C.c_int64(0)
    G = x.shape[0]
    b = _f64(bowl) if bowl is not None else None
    lib().or_adadelta(prob.ref() if prob is not None else None,
                      _p(b, C.c_double) if b is not None else None, G, C.byref(pp), iters,
                      _p(x, C.c_double), C.byref(Ec), C.byref(ev))
    return x, Ec.value, ev.value


def init_population(prob, pop, seed, ligand_id=0, run=0, energies=True):
    """D8 generation 0 of one run: (genes [pop, G], E [pop] or None)."""
    g = np.zeros((pop, prob.G)); E = np.zeros(pop) if energies else None
    lib().or_init_population(prob.ref(), pop, seed, ligand_id, run, _p(g, C.c_double),
                             _p(E, C.c_double) if energies else None)
    return g, E


def dock_run(prob, pp, pop, max_evals, seed, ligand_id=0, run=0):
    """One independent run (D8 + D11).  ctypes releases the GIL, so runs may be
    spread over Python threads to use several host cores."""
    bE = C.c_double(0); bg = np.zeros(prob.G); ev = C.c_int64(0); gens = C.c_int(0)
    fE = np.zeros(pop)
    lib().or_dock_run(prob.ref(), C.byref(pp), pop, max_evals, seed, ligand_id, run, C.byref(bE),
                      _p(bg, C.c_double), C.byref(ev), C.byref(gens), _p(fE, C.c_double))
    return dict(best_E=bE.value, best_genes=bg, evals=ev.value, generations=gens.value, final_E=fE)


def sum_evals(counters):
    c = np.ascontiguousarray(counters, dtype=np.int64)
    return int(lib().or_sum_evals(c.shape[0], _p(c, C.c_int64)))


# ---------------------------------------------------------------------------
# NEXT-3: clustering of per-run best poses
# ---------------------------------------------------------------------------
def rmsd(a, b):
    a = _f64(a).reshape(-1); b = _f64(b).reshape(-1)
    return float(lib().or_rmsd(a.shape[0] // 3, _p(a, C.c_double), _p(b, C.c_double)))


def cluster(xyz, E, rmsd_tol=2.0):
    """(n_clusters, cluster [n], rmsd_to_seed [n], rank [n]) of poses xyz [n, N, 3]."""
    x = _f64(xyz)
    n = x.shape[0]; N = x.shape[1] if x.ndim == 3 else x.reshape(n, -1).shape[1] // 3
    e = _f64(E)
    c = np.zeros(max(n, 1), np.int32); r = np.zeros(max(n, 1)); rk = np.zeros(max(n, 1), np.int32)
    nc = lib().or_cluster(n, N, _p(x, C.c_double), _p(e, C.c_double), float(rmsd_tol), _p(c, C.c_int),
                          _p(r, C.c_double), _p(rk, C.c_int))
    return int(nc), c[:n], r[:n], rk[:n]
