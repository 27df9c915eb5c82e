"""Python binding of libdock.so (include/dock.h): argument marshalling only.

Every step of the docking hot path (pose, grid interpolation, pair energy, gradient,
ADADELTA / Solis-Wets, GA, Philox) runs in the sm_100a kernels of libdock.so.  There is
no CPU fallback: importing this package fails loudly when the library is missing, and
every compute call raises when no CUDA device is usable.  PyTorch is used only for
device memory and streams (the *_device entry points accept torch CUDA tensors).
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# DOCK_LIB selects an experimental in-tree build variant (scripts/variants.py); default: the product library.
LIB_PATH = os.environ.get("DOCK_LIB") or os.path.join(_HERE, "libdock.so")

DOCK_OK, DOCK_E_INPUT, DOCK_E_INTERNAL = 0, 1, 2
LS_ADADELTA, LS_SOLIS_WETS = 0, 1
SF_D5, SF_AD4 = 0, 1          # dock_params.scoring (NEXT-2: D5-AD4)
PURPOSE_INIT, PURPOSE_GA, PURPOSE_LS_PICK, PURPOSE_SW = 0, 1, 2, 3


class DockError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"dock error {code}: {msg}")
        self.code = code


class Grids(C.Structure):
    _fields_ = [("nx", C.c_int32), ("ny", C.c_int32), ("nz", C.c_int32), ("spacing", C.c_float),
                ("origin", C.c_float * 3), ("n_types", C.c_int32), ("maps", C.POINTER(C.c_float)),
                ("type_names", C.POINTER(C.c_char * 4))]


class TypeParam(C.Structure):
    _fields_ = [("R", C.c_float), ("eps", C.c_float), ("S", C.c_float), ("V", C.c_float), ("role", C.c_int32)]


class Ligand(C.Structure):
    _fields_ = [("n_atoms", C.c_int32), ("type", C.POINTER(C.c_int32)), ("charge", C.POINTER(C.c_float)),
                ("xyz", C.POINTER(C.c_float)), ("n_bonds", C.c_int32), ("bonds", C.POINTER(C.c_int32)),
                ("rotatable", C.POINTER(C.c_uint8)), ("n_tors", C.c_int32), ("tors_axis", C.POINTER(C.c_int32)),
                ("tors_moved_off", C.POINTER(C.c_int32)), ("tors_moved", C.POINTER(C.c_int32)),
                ("n_pairs", C.c_int32), ("pairs", C.POINTER(C.c_int32))]


def _ligand_struct(types, charges, xyz, bonds, rotatable, tors=None, pairs=None):
    """A dock_ligand over numpy copies (returned alongside, to keep them alive).
    tors = (axis [T, 2], moved: T index lists) and pairs [P, 2]: verbatim topology (D1.7,
    SPEC TORSION / PAIR records); None: derived by D1 (n_tors = n_pairs = -1)."""
    t = np.ascontiguousarray(types, dtype=np.int32)
    q = np.ascontiguousarray(charges, dtype=np.float32)
    x = np.ascontiguousarray(xyz, dtype=np.float32).reshape(-1)
    b = np.ascontiguousarray(bonds if bonds is not None else np.zeros((0, 2)), dtype=np.int32).reshape(-1)
    r = np.ascontiguousarray(rotatable if rotatable is not None else np.zeros(b.shape[0] // 2), dtype=np.uint8)
    lg = Ligand()
    lg.n_atoms = t.shape[0]; lg.type = _ptr(t, C.c_int32); lg.charge = _ptr(q, C.c_float)
    lg.xyz = _ptr(x, C.c_float); lg.n_bonds = b.shape[0] // 2
    lg.bonds = _ptr(b, C.c_int32) if lg.n_bonds else None
    lg.rotatable = _ptr(r, C.c_uint8) if lg.n_bonds else None
    keep = [t, q, x, b, r]
    lg.n_tors = lg.n_pairs = -1
    if tors is not None or pairs is not None:
        axis, moved = tors if tors is not None else (np.zeros((0, 2)), [])
        ax = np.ascontiguousarray(axis, dtype=np.int32).reshape(-1)
        off = np.ascontiguousarray(np.concatenate([[0], np.cumsum([len(m) for m in moved])]), dtype=np.int32)
        mv = np.ascontiguousarray(np.concatenate([np.asarray(m, np.int64) for m in moved]) if len(moved) else
                                  np.zeros(0), dtype=np.int32)
        pr = np.ascontiguousarray(pairs if pairs is not None else np.zeros((0, 2)), dtype=np.int32).reshape(-1)
        keep += [ax, off, mv, pr]
        lg.n_tors = ax.shape[0] // 2
        lg.tors_axis = _ptr(ax, C.c_int32); lg.tors_moved_off = _ptr(off, C.c_int32); lg.tors_moved = _ptr(mv, C.c_int32)
        lg.n_pairs = pr.shape[0] // 2
        lg.pairs = _ptr(pr, C.c_int32)
    return lg, keep


def _names_array(type_names):
    """grids.type_names: [n_types] char[4] (NUL-terminated names), or None."""
    if type_names is None:
        return None
    arr = ((C.c_char * 4) * len(type_names))()
    for i, nm in enumerate(type_names):
        b = nm.encode() if isinstance(nm, str) else bytes(nm)
        if not 0 < len(b) < 4:
            raise DockError(DOCK_E_INPUT, f"type_names[{i}]: 1..3 characters")
        arr[i].value = b
    return arr


class Params(C.Structure):
    _fields_ = [("p_tour", C.c_float), ("p_cross", C.c_float), ("p_mut", C.c_float),
                ("mut_trans", C.c_float), ("mut_angle", C.c_float), ("ls_method", C.c_int32),
                ("ls_rate", C.c_float), ("ls_max_iters", C.c_int32), ("sw_rho", C.c_float),
                ("sw_rho_min", C.c_float), ("sw_expand", C.c_float), ("sw_contract", C.c_float),
                ("sw_cons_succ", C.c_int32), ("sw_cons_fail", C.c_int32), ("ad_rho", C.c_float),
                ("ad_eps", C.c_float), ("max_generations", C.c_int32), ("device", C.c_int32),
                ("l2_persist", C.c_int32), ("gens_per_graph", C.c_int32), ("profile", C.c_int32), ("sw_depth", C.c_int32),
                ("sw_split", C.c_int32), ("scoring", C.c_int32), ("w_vdw", C.c_float), ("w_hb", C.c_float),
                ("w_el", C.c_float), ("w_ds", C.c_float), ("w_tors", C.c_float), ("qasp", C.c_float),
                ("run_branches", C.c_int32)]


class ScreenOpts(C.Structure):
    _fields_ = [("n_devices", C.c_int32), ("devices", C.POINTER(C.c_int32)), ("slots_per_device", C.c_int32),
                ("prep_threads", C.c_int32)]


class ScreenStats(C.Structure):
    _fields_ = [("prep_ms", C.c_double), ("dock_ms", C.c_double), ("total_evals", C.c_int64),
                ("n_failed", C.c_int32), ("launches", C.c_int64)]


class ResultView(C.Structure):
    _fields_ = [("n_runs", C.c_int32), ("n_atoms", C.c_int32), ("n_genes", C.c_int32),
                ("best_energy", C.POINTER(C.c_float)), ("best_genotype", C.POINTER(C.c_float)),
                ("best_xyz", C.POINTER(C.c_float)), ("evals", C.POINTER(C.c_int64)),
                ("generations", C.POINTER(C.c_int32)), ("cluster", C.POINTER(C.c_int32)),
                ("rmsd_to_seed", C.POINTER(C.c_float)), ("dG", C.POINTER(C.c_float)),
                ("n_timings", C.c_int32), ("timing_names", C.POINTER(C.c_char_p)),
                ("timing_ms", C.POINTER(C.c_double))]


FMT_JSON, FMT_CSV = 0, 1
MAX_GENES = 38


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                          "g.build()'` (there is no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    P, v = C.POINTER, C.c_void_p
    i32, i64, u32, u64, f = C.c_int32, C.c_int64, C.c_uint32, C.c_uint64, C.c_float
    sig = {
        "dock_params_default": (i32, [P(Params)]),
        "dock_builtin_type_param": (i32, [C.c_char_p, P(TypeParam)]),
        "dock_init": (i32, [P(Grids), P(TypeParam), P(Ligand), P(Params), P(v)]),
        "dock_free": (None, [v]),
        "dock_last_error": (C.c_char_p, [v]),
        "dock_n_atoms": (i32, [v]), "dock_n_torsions": (i32, [v]),
        "dock_n_genes": (i32, [v]), "dock_n_pairs": (i32, [v]),
        "dock_run": (i32, [v, i32, i32, i64, u64, P(f), P(f), P(f), P(i64), P(i32)]),
        "dock_run_ex": (i32, [v, i32, i32, i32, u32, i64, u64, P(f), P(f), P(f), P(i64), P(i32)]),
        "dock_run_device": (i32, [v, i32, i32, i32, u32, i64, u64, v, v, v, v, v]),
        "dock_eval": (i32, [v, i32, P(f), P(f), P(f), P(f)]),
        "dock_eval_device": (i32, [v, i32, v, v, v, v, v]),
        "dock_eval_terms": (i32, [v, i32, P(f), P(f), P(f), P(f)]),
        "dock_cluster": (i32, [v, i32, P(f), P(f), f, P(i32), P(f), P(i32), P(i32)]),
        "dock_write_result": (i32, [P(ResultView), i32, C.c_char_p, C.c_size_t, P(C.c_size_t)]),
        "dock_write_screen": (i32, [i32, P(u32), P(f), P(i32), P(f), P(i32), P(i64), P(i32), P(i32), i32, C.c_char_p,
                                    C.c_size_t, P(C.c_size_t)]),
        "dock_bench_part": (i32, [v, i32, i32, i32, v, v, v]),
        "dock_get_pairs": (i32, [v, P(i32)]),
        "dock_get_torsions": (i32, [v, P(i32), P(C.c_uint8)]),
        "dock_philox": (i32, [i32, P(u32), P(u32), P(u32)]),
        "dock_stream_words": (i32, [u64, u32, u32, u32, u32, u32, u32, i32, P(u32)]),
        "dock_ga_step": (i32, [v, u64, u32, i32, i32, i32, P(f), P(f), P(f), P(f), P(i32), P(i32)]),
        "dock_init_population": (i32, [v, i32, i32, i32, u32, u64, P(f), P(f)]),
        "dock_bench_l2_gather": (i32, [i32, i32, i32, i32, P(C.c_double), P(C.c_double)]),
        "dock_ad_trace": (i32, [v, i32, i32, P(f), P(f), P(f), P(i64), P(f), P(f), P(f)]),
        "dock_sw_trace": (i32, [v, i32, i32, u64, u32, i32, i32, P(i32), P(f), P(f), P(f), P(i64), P(i32), P(f)]),
        "dock_ls_step": (i32, [v, i32, i32, i32, u64, u32, i32, i32, P(i32), P(f), P(f), P(i64)]),
        "dock_launch_count": (i64, [v]),
        "dock_kernel_stats": (i32, [v, P(C.c_double), P(i64)]),
        "dock_upload_bytes": (i64, [v]),
        "dock_run_branches": (i32, [v]),
        "dock_last_engine": (i32, [v]),
        "dock_tile_schedule": (i32, [v]),
        "dock_screen": (i32, [P(Grids), P(TypeParam), P(Ligand), i32, P(u32), P(Params), P(ScreenOpts), i32, i32,
                              i64, u64, P(f), P(i32), P(f), P(i64), P(i32), P(i32), P(ScreenStats)]),
        "dock_screen_last_error": (C.c_char_p, []),
        "dock_topology": (i32, [P(Ligand), P(TypeParam), i32, P(i32), P(i32), P(C.c_uint8), P(i32), P(i32), i32]),
    }
    for name, (res, args) in sig.items():
        if os.environ.get("DOCK_LIB") and not hasattr(L, name):
            continue                # experimental older build (A/B timing): symbol absent
        fn = getattr(L, name)
        fn.restype = res
        fn.argtypes = args
    return L


lib = _load()
EXPORTED = ("dock_params_default", "dock_builtin_type_param", "dock_init", "dock_free", "dock_last_error",
            "dock_n_atoms", "dock_n_torsions", "dock_n_genes", "dock_n_pairs", "dock_run", "dock_run_ex",
            "dock_run_device", "dock_eval", "dock_eval_device", "dock_get_pairs", "dock_get_torsions",
            "dock_philox", "dock_stream_words", "dock_ga_step", "dock_ls_step", "dock_launch_count",
            "dock_topology", "dock_kernel_stats", "dock_upload_bytes", "dock_screen", "dock_screen_last_error",
            "dock_bench_part", "dock_eval_terms", "dock_cluster", "dock_write_result", "dock_run_branches",
            "dock_write_screen", "dock_last_engine", "dock_init_population", "dock_sw_trace",
            "dock_ad_trace", "dock_bench_l2_gather", "dock_tile_schedule")


def write_result(res: dict, fmt: str = "json", timings: dict | None = None) -> str:
    """dock_write_result (NEXT-3): res has best_E [R], best_genes [R, G] and optionally
    best_xyz [R, N, 3], evals, generations, cluster, rmsd_to_seed, dG (arrays over runs)."""
    keep = []

    def arr(key, dt, ct):
        v = res.get(key)
        if v is None:
            return None
        a = np.ascontiguousarray(v, dtype=dt)
        keep.append(a)
        return _ptr(a, ct)
    bE = np.ascontiguousarray(res["best_E"], dtype=np.float32)
    bG = np.ascontiguousarray(res["best_genes"], dtype=np.float32)
    bG = bG.reshape(bE.shape[0], bG.shape[-1] if bG.ndim > 1 else -1)
    keep += [bE, bG]
    r = ResultView()
    r.n_runs = bE.shape[0]; r.n_genes = bG.shape[1]
    xyz = res.get("best_xyz")
    r.n_atoms = 0 if xyz is None else int(np.asarray(xyz).shape[1])
    r.best_energy = _ptr(bE, C.c_float); r.best_genotype = _ptr(bG, C.c_float)
    r.best_xyz = arr("best_xyz", np.float32, C.c_float)
    r.evals = arr("evals", np.int64, C.c_int64)
    r.generations = arr("generations", np.int32, C.c_int32)
    r.cluster = arr("cluster", np.int32, C.c_int32)
    r.rmsd_to_seed = arr("rmsd_to_seed", np.float32, C.c_float)
    r.dG = arr("dG", np.float32, C.c_float)
    timings = timings or {}
    names = (C.c_char_p * max(1, len(timings)))(*[k.encode() for k in timings])
    ms = np.ascontiguousarray(list(timings.values()) or [0.0], dtype=np.float64)
    r.n_timings = len(timings); r.timing_names = names; r.timing_ms = _ptr(ms, C.c_double)
    f = {"json": FMT_JSON, "csv": FMT_CSV}[fmt]
    need = C.c_size_t(0)
    lib.dock_write_result(C.byref(r), f, None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    _check(lib.dock_write_result(C.byref(r), f, buf, need.value, C.byref(need)))
    return buf.value.decode()


def write_screen(out: dict, fmt: str = "json", ids=None, n_genes=None) -> str:
    """dock_write_screen (NEXT-3): a screen() result dict -> JSON / CSV text."""
    bE = np.ascontiguousarray(out["best_E"], dtype=np.float32)
    n = bE.shape[0]
    keep = []

    def arr(v, dt, ct):
        if v is None:
            return None
        a = np.ascontiguousarray(v, dtype=dt)
        keep.append(a)
        return _ptr(a, ct)
    f = {"json": FMT_JSON, "csv": FMT_CSV}[fmt]
    args = [n, arr(ids, np.uint32, C.c_uint32), _ptr(bE, C.c_float), arr(out.get("best_run"), np.int32, C.c_int32),
            arr(out.get("best_genes"), np.float32, C.c_float), arr(n_genes, np.int32, C.c_int32),
            arr(out.get("evals"), np.int64, C.c_int64), arr(out.get("status"), np.int32, C.c_int32),
            arr(out.get("device"), np.int32, C.c_int32), f]
    need = C.c_size_t(0)
    lib.dock_write_screen(*args, None, 0, C.byref(need))
    buf = C.create_string_buffer(need.value)
    rc = lib.dock_write_screen(*args, buf, need.value, C.byref(need))
    if rc != DOCK_OK:
        raise DockError(rc, "dock_write_screen")
    return buf.value.decode()


def topology(types, charges, xyz, bonds, rotatable, type_params, roles, tors=None, pairs=None):
    """D1 on the host (no device needed): (axis [T,2], moved [T,N], pairs [P,2]).  tors /
    pairs: verbatim topology to validate (D1.7), as in Docker."""
    tp = np.asarray(type_params, dtype=np.float32).reshape(-1, 4)
    tarr = (TypeParam * tp.shape[0])()
    for k in range(tp.shape[0]):
        tarr[k] = TypeParam(*(float(v) for v in tp[k]), int(roles[k]))
    lg, keep = _ligand_struct(types, charges, xyz, bonds, rotatable, tors, pairs)
    N = lg.n_atoms
    cap = max(1, N * (N - 1) // 2)
    T = C.c_int32(0); Pn = C.c_int32(0)
    axis = np.zeros(64, np.int32); moved = np.zeros(32 * N, np.uint8); pairs_out = np.zeros(2 * cap, np.int32)
    _check(lib.dock_topology(C.byref(lg), tarr, tp.shape[0], C.byref(T), _ptr(axis, C.c_int32),
                             _ptr(moved, C.c_uint8), C.byref(Pn), _ptr(pairs_out, C.c_int32), cap))
    return (axis[: 2 * T.value].reshape(-1, 2), moved[: T.value * N].reshape(T.value, N),
            pairs_out[: 2 * Pn.value].reshape(-1, 2))


def _ptr(a, ct):
    return a.ctypes.data_as(C.POINTER(ct)) if a is not None else None


def _check(rc, ctx=None):
    if rc != DOCK_OK:
        msg = lib.dock_last_error(ctx)
        raise DockError(rc, msg.decode() if msg else "")


def params_default(**overrides) -> Params:
    p = Params()
    _check(lib.dock_params_default(C.byref(p)))
    for k, val in overrides.items():
        if not hasattr(p, k):
            raise KeyError(k)
        setattr(p, k, val)
    return p


def builtin_type_param(name: str) -> TypeParam:
    t = TypeParam()
    _check(lib.dock_builtin_type_param(name.encode(), C.byref(t)))
    return t


def bench_l2_gather(device=0, mib=48, blocks_per_sm=8, iters=64):
    """L2 gather ceiling (dock_bench_l2_gather): (GB/s of random 16-byte loads, ms)."""
    g = C.c_double(0); t = C.c_double(0)
    _check(lib.dock_bench_l2_gather(device, mib, blocks_per_sm, iters, C.byref(g), C.byref(t)))
    return g.value, t.value


def philox(ctr, key):
    """Raw Philox4x32-10 on the device: ctr [n,4] u32, key [n,2] u32 -> [n,4]."""
    c = np.ascontiguousarray(ctr, dtype=np.uint32).reshape(-1, 4)
    k = np.ascontiguousarray(key, dtype=np.uint32).reshape(-1, 2)
    out = np.zeros_like(c)
    _check(lib.dock_philox(c.shape[0], _ptr(c, C.c_uint32), _ptr(k, C.c_uint32), _ptr(out, C.c_uint32)))
    return out


def stream_words(seed, ligand_id, purpose, slot, gen, run, m0, n):
    out = np.zeros(n, np.uint32)
    _check(lib.dock_stream_words(seed, ligand_id, purpose, slot, gen, run, m0, n, _ptr(out, C.c_uint32)))
    return out


def _grids_struct(maps, n, spacing, origin, n_types):
    g = Grids()
    g.nx, g.ny, g.nz = (int(v) for v in n)
    g.spacing = float(spacing)
    for d in range(3):
        g.origin[d] = float(origin[d])
    g.n_types = int(n_types)
    g.maps = _ptr(maps, C.c_float)
    return g


def _type_array(type_params, roles):
    tp = np.asarray(type_params, dtype=np.float32).reshape(-1, 4)
    roles = np.asarray(roles, dtype=np.int32).reshape(-1)
    tarr = (TypeParam * tp.shape[0])()
    for t in range(tp.shape[0]):
        tarr[t] = TypeParam(*(float(x) for x in tp[t]), int(roles[t]))
    return tarr, tp.shape[0]


def screen(grid, ligands, pop, runs, max_evals, seed, ligand_ids=None, devices=None, slots_per_device=0,
           prep_threads=0, params: Params | None = None, **overrides):
    """dock_screen (include/dock.h): dock every ligand against one receptor on the given
    CUDA devices.  grid: gen.synth-like object (maps/n/spacing/origin/type_params());
    ligands: objects with types/charges/xyz/bonds/rotatable.  Returns a dict of per-ligand
    arrays (best_E, best_run, best_genes [n, 38] zero padded, evals, status, device) and
    the screen stats."""
    maps = np.ascontiguousarray(grid.maps, dtype=np.float32).reshape(-1)
    tp, roles = grid.type_params()
    tarr, nt = _type_array(tp, roles)
    g = _grids_struct(maps, grid.n, grid.spacing, grid.origin, nt)
    n = len(ligands)
    keep = []
    larr = (Ligand * max(n, 1))()
    for i, lig in enumerate(ligands):
        lg, kp = _ligand_struct(lig.types, lig.charges, lig.xyz, lig.bonds, lig.rotatable,
                                getattr(lig, "tors", None), getattr(lig, "pairs", None))
        keep.append(kp)
        larr[i] = lg
    ids = None if ligand_ids is None else np.ascontiguousarray(ligand_ids, dtype=np.uint32)
    if params is None:
        params = params_default(**overrides)
    else:
        for k, val in overrides.items():
            setattr(params, k, val)
    o = ScreenOpts()
    dv = None
    if devices is not None:
        dv = np.ascontiguousarray(devices, dtype=np.int32)
        o.n_devices = dv.shape[0]; o.devices = _ptr(dv, C.c_int32)
    o.slots_per_device = int(slots_per_device); o.prep_threads = int(prep_threads)
    out = dict(best_E=np.zeros(n, np.float32), best_run=np.zeros(n, np.int32),
               best_genes=np.zeros((n, MAX_GENES), np.float32), evals=np.zeros(n, np.int64),
               status=np.zeros(n, np.int32), device=np.zeros(n, np.int32))
    st = ScreenStats()
    rc = lib.dock_screen(C.byref(g), tarr, larr, n, _ptr(ids, C.c_uint32), C.byref(params), C.byref(o), pop, runs,
                         max_evals, seed, _ptr(out["best_E"], C.c_float), _ptr(out["best_run"], C.c_int32),
                         _ptr(out["best_genes"], C.c_float), _ptr(out["evals"], C.c_int64),
                         _ptr(out["status"], C.c_int32), _ptr(out["device"], C.c_int32), C.byref(st))
    if rc != DOCK_OK:
        msg = lib.dock_screen_last_error()
        raise DockError(rc, msg.decode() if msg else "")
    out["stats"] = dict(prep_ms=st.prep_ms, dock_ms=st.dock_ms, total_evals=st.total_evals, n_failed=st.n_failed,
                        launches=st.launches)
    return out


class Docker:
    """One (device, receptor grid, ligand) docking context (dock_init ... dock_free)."""

    def __init__(self, maps, n, spacing, origin, type_params, roles, types, charges, xyz, bonds,
                 rotatable, params: Params | None = None, tors=None, pairs=None, type_names=None, **overrides):
        """type_params None: the built-in table by type_names (dock_init with NULL type_params);
        tors = (axis [T, 2], moved index lists) and / or pairs [P, 2]: verbatim topology."""
        maps = np.ascontiguousarray(maps, dtype=np.float32).reshape(-1)
        n = tuple(int(v) for v in n)
        g = Grids()
        g.nx, g.ny, g.nz = n
        g.spacing = float(spacing)
        for d in range(3):
            g.origin[d] = float(origin[d])
        g.maps = _ptr(maps, C.c_float)
        self._names = _names_array(type_names)
        g.type_names = C.cast(self._names, C.POINTER(C.c_char * 4)) if self._names is not None else None
        if type_params is None:
            if type_names is None:
                raise DockError(DOCK_E_INPUT, "type_params None needs type_names (the built-in table)")
            g.n_types = len(type_names)
            tarr = None
        else:
            tp = np.asarray(type_params, dtype=np.float32).reshape(-1, 4)
            roles = np.asarray(roles, dtype=np.int32).reshape(-1)
            g.n_types = tp.shape[0]
            tarr = (TypeParam * tp.shape[0])()
            for t in range(tp.shape[0]):
                tarr[t] = TypeParam(*(float(x) for x in tp[t]), int(roles[t]))
        lg, self._keep = _ligand_struct(types, charges, xyz, bonds, rotatable, tors, pairs)
        if params is None:
            params = params_default(**overrides)
        else:
            for k, val in overrides.items():
                setattr(params, k, val)
        self.params = params
        self._ctx = C.c_void_p()
        _check(lib.dock_init(C.byref(g), tarr, C.byref(lg), C.byref(params), C.byref(self._ctx)))
        self.N = lib.dock_n_atoms(self._ctx)
        self.T = lib.dock_n_torsions(self._ctx)
        self.G = lib.dock_n_genes(self._ctx)
        self.P = lib.dock_n_pairs(self._ctx)

    @classmethod
    def from_inputs(cls, grid, lig, params: Params | None = None, **overrides):
        """Duck-typed constructor: grid has maps/n/spacing/origin/type_params(); lig has
        types/charges/xyz/bonds/rotatable (e.g. gen.synth objects)."""
        tp, roles = grid.type_params()
        return cls(grid.maps, grid.n, grid.spacing, grid.origin, tp, roles, lig.types, lig.charges,
                   lig.xyz, lig.bonds, lig.rotatable, params=params, **overrides)

    def close(self):
        if getattr(self, "_ctx", None) and self._ctx.value:
            lib.dock_free(self._ctx)
            self._ctx = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _chk(self, rc):
        _check(rc, self._ctx)

    @property
    def launches(self) -> int:
        return int(lib.dock_launch_count(self._ctx))

    @property
    def run_branches(self) -> int:
        """Concurrent run branches of the last run (1 = lockstep generations)."""
        return int(lib.dock_run_branches(self._ctx))

    ENGINES = ("lockstep", "branches", "clusters")

    @property
    def engine(self) -> str:
        """Generation engine of the last run (dock_last_engine): lockstep, branches or clusters."""
        return self.ENGINES[int(lib.dock_last_engine(self._ctx))]

    @property
    def tile_schedule(self) -> dict:
        """Gradient pair-tile schedule of this ligand (dock_tile_schedule)."""
        v = int(lib.dock_tile_schedule(self._ctx))
        return {"slots": bool(v & 1), "tail": ("rot" if v & 2 else "seg" if v & 4 else "hyb" if v & 8 else "bcast"),
                "packed": bool(v & 16), "hb_side_pairs": (v >> 8) & 0xff}

    @property
    def upload_bytes(self) -> int:
        return int(lib.dock_upload_bytes(self._ctx))

    def kernel_stats(self):
        """(ms[3], launches[3]) for kernel classes (k_ga, k_ls_*, k_init) of the last run
        (needs profile=1)."""
        ms = np.zeros(3, np.float64); n = np.zeros(3, np.int64)
        self._chk(lib.dock_kernel_stats(self._ctx, _ptr(ms, C.c_double), _ptr(n, C.c_int64)))
        return ms, n

    # ---- D1 ----
    def pairs(self):
        out = np.zeros(max(1, 2 * self.P), np.int32)
        self._chk(lib.dock_get_pairs(self._ctx, _ptr(out, C.c_int32)))
        return out[: 2 * self.P].reshape(-1, 2)

    def torsions(self):
        axis = np.zeros(max(1, 2 * self.T), np.int32)
        moved = np.zeros(max(1, self.T * self.N), np.uint8)
        self._chk(lib.dock_get_torsions(self._ctx, _ptr(axis, C.c_int32), _ptr(moved, C.c_uint8)))
        return axis[: 2 * self.T].reshape(-1, 2), moved[: self.T * self.N].reshape(self.T, self.N)

    # ---- D3-D7 ----
    def eval(self, genotypes, grad=False, xyz=False):
        x = np.ascontiguousarray(genotypes, dtype=np.float32).reshape(-1, self.G)
        n = x.shape[0]
        E = np.zeros(n, np.float32)
        gr = np.zeros((n, self.G), np.float32) if grad else None
        xy = np.zeros((n, self.N, 3), np.float32) if xyz else None
        self._chk(lib.dock_eval(self._ctx, n, _ptr(x, C.c_float), _ptr(E, C.c_float), _ptr(gr, C.c_float),
                                _ptr(xy, C.c_float)))
        return E, gr, xy

    def eval_terms(self, genotypes):
        """(inter [n], intra [n], dG [n]) through dock_eval_terms (dG = inter + w_tors T)."""
        x = np.ascontiguousarray(genotypes, dtype=np.float32).reshape(-1, self.G)
        n = x.shape[0]
        out = [np.zeros(n, np.float32) for _ in range(3)]
        self._chk(lib.dock_eval_terms(self._ctx, n, _ptr(x, C.c_float), *(_ptr(o, C.c_float) for o in out)))
        return tuple(out)

    # ---- NEXT-3 ----
    def cluster(self, xyz, energy, rmsd_tol=2.0):
        """dock_cluster: (n_clusters, cluster [n], rmsd_to_seed [n], rank [n]) of poses [n, N, 3]."""
        x = np.ascontiguousarray(xyz, dtype=np.float32).reshape(-1, self.N, 3)
        e = np.ascontiguousarray(energy, dtype=np.float32).reshape(-1)
        n = x.shape[0]
        c = np.zeros(max(n, 1), np.int32); r = np.zeros(max(n, 1), np.float32); rk = np.zeros(max(n, 1), np.int32)
        nc = C.c_int32(0)
        self._chk(lib.dock_cluster(self._ctx, n, _ptr(x, C.c_float), _ptr(e, C.c_float), float(rmsd_tol),
                                   _ptr(c, C.c_int32), _ptr(r, C.c_float), _ptr(rk, C.c_int32), C.byref(nc)))
        return int(nc.value), c[:n], r[:n], rk[:n]

    def eval_device(self, genotypes, energy, grad=None, xyz=None, stream=0):
        """torch CUDA tensors (float32, contiguous); stream = torch.cuda.Stream.cuda_stream or 0."""
        n = genotypes.shape[0]
        self._chk(lib.dock_eval_device(self._ctx, n, genotypes.data_ptr(), energy.data_ptr(),
                                       grad.data_ptr() if grad is not None else None,
                                       xyz.data_ptr() if xyz is not None else None, stream or None))

    def bench_part(self, part, genotypes, out, iters, stream=0):
        """Microbenchmark (dock_bench_part): part 0 = pose + grid interpolation, 1 = pose +
        pair tiles; torch CUDA tensors genotypes [n, G] and out [n]."""
        self._chk(lib.dock_bench_part(self._ctx, part, genotypes.shape[0], iters, genotypes.data_ptr(),
                                      out.data_ptr(), stream or None))

    # ---- D8-D11 ----
    def run(self, pop, runs, max_evals, seed, run_base=0, ligand_id=0, xyz=True):
        bE = np.zeros(runs, np.float32)
        bG = np.zeros((runs, self.G), np.float32)
        bX = np.zeros((runs, self.N, 3), np.float32) if xyz else None
        ev = np.zeros(runs, np.int64)
        gens = np.zeros(runs, np.int32)
        self._chk(lib.dock_run_ex(self._ctx, pop, runs, run_base, ligand_id, max_evals, seed,
                                  _ptr(bE, C.c_float), _ptr(bG, C.c_float), _ptr(bX, C.c_float),
                                  _ptr(ev, C.c_int64), _ptr(gens, C.c_int32)))
        return dict(best_E=bE, best_genes=bG, best_xyz=bX, evals=ev, generations=gens)

    def _check_dev(self, name, t, dtype, numel):
        """A device output buffer the kernels write: right dtype, on this context's device,
        contiguous and large enough (DockError otherwise, before any launch)."""
        import torch
        if not isinstance(t, torch.Tensor):
            raise DockError(DOCK_E_INPUT, f"{name}: expected a torch CUDA tensor")
        if t.dtype != dtype or not t.is_cuda or t.device.index != self.params.device or not t.is_contiguous() \
                or t.numel() < numel:
            raise DockError(DOCK_E_INPUT, f"{name}: need a contiguous {dtype} tensor on cuda:{self.params.device} "
                                          f"with >= {numel} elements (got {t.dtype}, {t.device}, {t.numel()})")

    def run_device(self, pop, runs, max_evals, seed, best_E, best_genes, evals=None, gens=None,
                   run_base=0, ligand_id=0, stream=0):
        import torch
        self._check_dev("best_E", best_E, torch.float32, runs)
        self._check_dev("best_genes", best_genes, torch.float32, runs * self.G)
        if evals is not None:
            self._check_dev("evals", evals, torch.int64, runs)
        if gens is not None:
            self._check_dev("gens", gens, torch.int32, runs)
        self._chk(lib.dock_run_device(self._ctx, pop, runs, run_base, ligand_id, max_evals, seed,
                                      best_E.data_ptr(), best_genes.data_ptr(),
                                      evals.data_ptr() if evals is not None else None,
                                      gens.data_ptr() if gens is not None else None, stream or None))

    def init_population(self, pop, runs, seed, run_base=0, ligand_id=0):
        """Generation 0 as dock_run_ex draws it (row a2): genes [runs, pop, G], E [runs, pop]."""
        g = np.zeros((runs, pop, self.G), np.float32)
        E = np.zeros((runs, pop), np.float32)
        self._chk(lib.dock_init_population(self._ctx, pop, runs, run_base, ligand_id, seed, _ptr(g, C.c_float),
                                           _ptr(E, C.c_float)))
        return g, E

    def ga_step(self, seed, ligand_id, run, gen, old_genes, old_E):
        og = np.ascontiguousarray(old_genes, dtype=np.float32)
        oE = np.ascontiguousarray(old_E, dtype=np.float32)
        pop = og.shape[0]
        ng = np.zeros_like(og); nE = np.zeros_like(oE)
        dbg = np.zeros((pop, 8), np.int32); perm = np.zeros(pop, np.int32)
        self._chk(lib.dock_ga_step(self._ctx, seed, ligand_id, run, gen, pop, _ptr(og, C.c_float),
                                   _ptr(oE, C.c_float), _ptr(ng, C.c_float), _ptr(nE, C.c_float),
                                   _ptr(dbg, C.c_int32), _ptr(perm, C.c_int32)))
        return ng, nE, dbg, perm

    def sw_trace(self, genes, energy, iters, seed=0, ligand_id=0, run=0, gen=1, slots=None, fed=None):
        """Solis-Wets with traces (dock_sw_trace): fed [n, iters, 2] candidate energies or None.
        Returns genes, E, evals, outcome [n, iters] (-1 = not executed), rho [n, iters]."""
        g = np.ascontiguousarray(genes, dtype=np.float32).reshape(-1, self.G).copy()
        E = np.ascontiguousarray(energy, dtype=np.float32).copy()
        n = g.shape[0]
        sl = np.ascontiguousarray(slots if slots is not None else np.arange(n), dtype=np.int32)
        fd = np.ascontiguousarray(fed, dtype=np.float32).reshape(n, iters, 2) if fed is not None else None
        ev = np.zeros(n, np.int64)
        to = np.zeros((n, iters), np.int32); tr = np.zeros((n, iters), np.float32)
        self._chk(lib.dock_sw_trace(self._ctx, n, iters, seed, ligand_id, run, gen, _ptr(sl, C.c_int32),
                                    _ptr(fd, C.c_float) if fd is not None else None, _ptr(g, C.c_float),
                                    _ptr(E, C.c_float), _ptr(ev, C.c_int64), _ptr(to, C.c_int32), _ptr(tr, C.c_float)))
        return g, E, ev, to, tr

    def ad_trace(self, genes, energy, iters, fed=None):
        """ADADELTA with traces (dock_ad_trace): fed [n, iters, 1+G] (energy, gradient) or None.
        Returns genes, E, evals, trace_x [n, iters, G], trace_E [n, iters], trace_g [n, iters, G]."""
        g = np.ascontiguousarray(genes, dtype=np.float32).reshape(-1, self.G).copy()
        E = np.ascontiguousarray(energy, dtype=np.float32).copy()
        n = g.shape[0]
        fd = np.ascontiguousarray(fed, dtype=np.float32).reshape(n, iters, self.G + 1) if fed is not None else None
        ev = np.zeros(n, np.int64)
        tx = np.zeros((n, iters, self.G), np.float32); tE = np.zeros((n, iters), np.float32)
        tg = np.zeros((n, iters, self.G), np.float32)
        self._chk(lib.dock_ad_trace(self._ctx, n, iters, _ptr(fd, C.c_float) if fd is not None else None,
                                    _ptr(g, C.c_float), _ptr(E, C.c_float), _ptr(ev, C.c_int64), _ptr(tx, C.c_float),
                                    _ptr(tE, C.c_float), _ptr(tg, C.c_float)))
        return g, E, ev, tx, tE, tg

    def ls_step(self, method, genes, energy, iters, seed=0, ligand_id=0, run=0, gen=1, slots=None):
        g = np.ascontiguousarray(genes, dtype=np.float32).reshape(-1, self.G).copy()
        E = np.ascontiguousarray(energy, dtype=np.float32).copy()
        n = g.shape[0]
        sl = np.ascontiguousarray(slots if slots is not None else np.arange(n), dtype=np.int32)
        ev = np.zeros(n, np.int64)
        self._chk(lib.dock_ls_step(self._ctx, method, n, iters, seed, ligand_id, run, gen, _ptr(sl, C.c_int32),
                                   _ptr(g, C.c_float), _ptr(E, C.c_float), _ptr(ev, C.c_int64)))
        return g, E, ev
