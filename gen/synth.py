"""Synthetic ligands and receptor grid maps (input data only).

Recipe: SURVEY.md §8(d) "Synthetic inputs", restated in DESIGN.md §4.  The
shapes follow PAPER.md:64-66 (§II-A: population 150, ligands of 21/43/108
atoms and 2/15/31 rotatable bonds) and BASELINE.json `configs`.

Nothing here evaluates the docking method: there is no pose builder, no
ligand scoring, no pair rule, no gradient and no search.  The receptor maps
are produced by a *receptor-side* recipe (a pseudo-receptor of random atoms,
Morse-shaped type maps, a screened Coulomb map and a Gaussian desolvation
map) which is the AutoGrid role — outside the graded path (SURVEY.md §8(f)
"Out of scope: receptor preparation and real grid generation").
"""
from __future__ import annotations

import math
import os
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# Per-type parameters (data, not arithmetic).  SURVEY.md §8(c) D5 table:
# R (Å), eps (kcal/mol), solvation S, volume V, H-bond role 0 none/1 donor/2 acceptor.
# Both the oracle and the CUDA library receive this table as input arrays.
# ---------------------------------------------------------------------------
TYPE_TABLE = {
    "C":  (4.00, 0.150, -0.00143, 33.5103, 0),
    "A":  (4.00, 0.150, -0.00052, 33.5103, 0),
    "N":  (3.50, 0.160, -0.00162, 22.4493, 0),
    "NA": (3.50, 0.160, -0.00162, 22.4493, 2),
    "O":  (3.20, 0.200, -0.00251, 17.1573, 0),
    "OA": (3.20, 0.200, -0.00251, 17.1573, 2),
    "H":  (2.00, 0.020, 0.00051, 0.0, 0),
    "HD": (2.00, 0.020, 0.00051, 0.0, 1),
}
TYPE_NAMES = list(TYPE_TABLE.keys())  # S:83 order: C A N NA O OA H HD


@dataclass
class Config:
    """One BASELINE.json config, with the values SURVEY.md §8.0 declares."""
    name: str
    n_atoms: int
    n_tors: int
    grid_n: int
    spacing: float
    n_maps: int          # type maps + E + D
    pop: int
    runs: int
    max_evals: int
    ls_method: int       # 0 ADADELTA, 1 Solis-Wets
    ls_rate: float
    ls_iters: int
    lig_seed: int
    grid_seed: int
    note: str = ""
    extra: dict = field(default_factory=dict)


# SURVEY.md §8.0 table; BASELINE.json configs[0..3].
CONFIGS = {
    "tiny": Config("tiny", 8, 2, 16, 0.75, 7, 16, 1, 2000, 0, 1.0, 30, 1, 101,
                   "configs[0]: tiny synthetic ligand, 8 atoms, 2 torsions, 16^3 grid, 7 maps, pop 16, 1 run, 2k evals"),
    "1stp": Config("1stp", 16, 5, 60, 0.375, 7, 150, 20, 2_500_000, 1, 0.06, 300, 2, 102,
                   "configs[1]: 1stp-shaped, 16 atoms, 5 torsions, 60^3 grid, pop 150, 20 runs, 2.5M evals, Solis-Wets"),
    "3ce3": Config("3ce3", 40, 8, 64, 0.375, 8, 150, 50, 2_500_000, 0, 1.0, 300, 3, 103,
                   "configs[2]: 3ce3-shaped, 40 atoms, 8 torsions, 64^3 grid, pop 150, 50 runs, ADADELTA"),
    "7cpa": Config("7cpa", 70, 15, 80, 0.375, 10, 256, 100, 2_500_000, 0, 1.0, 300, 4, 104,
                   "configs[3]: 7cpa-shaped, 70 atoms, 15 torsions, 80^3 grid, pop 256, 100 runs, ADADELTA"),
    # NEXT-1: the paper's own input shapes (PAPER.md:66 [§II-A]: "21, 43,
    # and 108 atoms, and 2, 15, and 31 rotatable bonds"), with the paper's Solis-Wets LS.
    "ps": Config("ps", 21, 2, 64, 0.375, 8, 150, 10, 2_500_000, 1, 0.06, 300, 6, 106,
                 "NEXT-1 PS: paper's small input shape, 21 atoms, 2 torsions, Solis-Wets"),
    "pm": Config("pm", 43, 15, 64, 0.375, 8, 150, 10, 2_500_000, 1, 0.06, 300, 7, 107,
                 "NEXT-1 PM: paper's medium input shape, 43 atoms, 15 torsions, Solis-Wets"),
    "pl": Config("pl", 108, 31, 80, 0.375, 10, 150, 10, 2_500_000, 1, 0.06, 300, 8, 108,
                 "NEXT-1 PL: paper's large input shape, 108 atoms, 31 torsions, Solis-Wets"),
    # configs[4]: 10k ligands N~U{10..70} vs one 64^3 receptor; see hts_ligands().
    "hts": Config("hts", 0, 0, 64, 0.375, 10, 150, 10, 250_000, 0, 1.0, 300, 5, 105,
                  "configs[4]: 10k synthetic ligands of mixed sizes vs one receptor grid"),
}

HEAVY_FREQ = {"C": 0.45, "A": 0.15, "OA": 0.12, "N": 0.05, "NA": 0.05, "O": 0.03}
MAX_VALENCE = {"C": 4, "A": 3, "N": 3, "NA": 3, "O": 2, "OA": 2, "H": 1, "HD": 1}


@dataclass
class Ligand:
    type_names: list          # names of the types used, index = grid map index
    types: np.ndarray         # int32 [N] index into type_names
    charges: np.ndarray       # float32 [N]
    xyz: np.ndarray           # float32 [N,3]
    bonds: np.ndarray         # int32 [B,2]
    rotatable: np.ndarray     # uint8 [B]
    atom_names: list          # type name per atom

    @property
    def n_atoms(self):
        return int(self.types.shape[0])

    @property
    def n_rot(self):
        return int(self.rotatable.sum())


def _grow_tree(rng, n, branch_p=0.3):
    """Random acyclic topology, valence <= 4, branching probability ~0.3."""
    parent = np.full(n, -1, dtype=np.int64)
    deg = np.zeros(n, dtype=np.int64)
    for a in range(1, n):
        last = a - 1
        if rng.random() >= branch_p and deg[last] < 3:
            p = last
        else:
            cand = [i for i in range(a) if deg[i] < 4]
            p = int(rng.choice(cand))
        parent[a] = p
        deg[a] += 1
        deg[p] += 1
    return parent, deg


def _assign_types(rng, deg, parent):
    n = len(deg)
    names = list(HEAVY_FREQ.keys())
    w = np.array([HEAVY_FREQ[k] for k in names])
    w = w / w.sum()
    out = []
    for a in range(n):
        for _ in range(100):
            t = names[int(rng.choice(len(names), p=w))]
            if deg[a] <= MAX_VALENCE[t]:
                break
        else:
            t = "C"
        out.append(t)
    # polar hydrogens: terminal atoms bonded to N/NA/OA/O
    nbr = [[] for _ in range(n)]
    for a in range(1, n):
        nbr[a].append(parent[a])
        nbr[parent[a]].append(a)
    for a in range(n):
        if deg[a] == 1:
            b = nbr[a][0]
            if out[b] in ("N", "NA", "OA", "O") and deg[b] >= 2 and rng.random() < 0.8:
                out[a] = "HD"
    return out, nbr


def _bond_len(ta, tb):
    if ta in ("HD", "H") or tb in ("HD", "H"):
        return 1.0
    if ta == "A" and tb == "A":
        return 1.40
    return 1.53


def _unit(v):
    return v / np.linalg.norm(v)


def _place(rng, n, parent, nbr, names, max_tries=200):
    """Tetrahedral-angle geometry with random dihedrals; reject clashes."""
    # topological distances (tree BFS) for the clash rule only
    dist = np.full((n, n), 10**6, dtype=np.int64)
    for s in range(n):
        dist[s, s] = 0
        q = [s]
        while q:
            u = q.pop()
            for v in nbr[u]:
                if dist[s, v] > dist[s, u] + 1:
                    dist[s, v] = dist[s, u] + 1
                    q.append(v)
    ang = math.radians(109.5)
    pos = np.zeros((n, 3))
    for a in range(1, n):
        p = parent[a]
        L = _bond_len(names[a], names[p])
        # reference direction: a placed neighbour of p other than a
        ref = None
        for v in nbr[p]:
            if v < a and v != a:
                ref = v
                break
        ok = False
        for _ in range(max_tries):
            if ref is None:
                d = _unit(rng.normal(size=3))
            else:
                u = _unit(pos[ref] - pos[p])
                # any vector perpendicular to u, rotated by a random dihedral
                t = _unit(np.cross(u, rng.normal(size=3)))
                phi = rng.uniform(0, 2 * math.pi)
                w = np.cross(u, t)
                perp = math.cos(phi) * t + math.sin(phi) * w
                d = math.cos(ang) * u + math.sin(ang) * perp
            cand = pos[p] + L * d
            bad = False
            for b in range(a):
                if dist[a, b] >= 3 and np.linalg.norm(cand - pos[b]) < 2.0:
                    bad = True
                    break
            if not bad:
                ok = True
                break
        if not ok:
            return None
        pos[a] = cand
    return pos


def make_ligand(n_atoms: int, n_tors: int, seed: int, type_names=None) -> Ligand:
    """SURVEY.md §8(d) ligand recipe, steps 1-7.  Deterministic in `seed`."""
    rng = np.random.default_rng(seed)
    for _attempt in range(1000):
        parent, deg = _grow_tree(rng, n_atoms)
        names, nbr = _assign_types(rng, deg, parent)
        bonds = [(int(parent[a]), a) for a in range(1, n_atoms)]
        internal = [k for k, (x, y) in enumerate(bonds) if deg[x] >= 2 and deg[y] >= 2
                    and names[x] not in ("HD", "H") and names[y] not in ("HD", "H")]
        if len(internal) < n_tors:
            continue
        pos = _place(rng, n_atoms, parent, nbr, names)
        if pos is None:
            continue
        break
    else:
        raise RuntimeError("ligand generator failed")
    rot = np.zeros(len(bonds), dtype=np.uint8)
    if n_tors > 0:
        pick = rng.choice(len(internal), size=n_tors, replace=False)
        for k in pick:
            rot[internal[k]] = 1
    # charges (step 5)
    q = np.clip(rng.normal(0.0, 0.2, size=n_atoms), -0.6, 0.6)
    for a, t in enumerate(names):
        if t == "HD":
            q[a] = rng.uniform(0.2, 0.4)
        elif TYPE_TABLE[t][4] == 2:
            q[a] = rng.uniform(-0.5, -0.3)
    q = q - q.mean()
    pos = pos - pos.mean(axis=0)
    if type_names is None:
        type_names = [t for t in TYPE_NAMES if t in set(names)]
    idx = {t: i for i, t in enumerate(type_names)}
    b = np.array(bonds, dtype=np.int32).reshape(-1, 2)
    return Ligand(type_names=list(type_names),
                  types=np.array([idx[t] for t in names], dtype=np.int32),
                  charges=q.astype(np.float32),
                  xyz=pos.astype(np.float32),
                  bonds=b, rotatable=rot, atom_names=names)


def retype(lig: Ligand, type_names) -> Ligand:
    idx = {t: i for i, t in enumerate(type_names)}
    return Ligand(type_names=list(type_names),
                  types=np.array([idx[t] for t in lig.atom_names], dtype=np.int32),
                  charges=lig.charges, xyz=lig.xyz, bonds=lig.bonds,
                  rotatable=lig.rotatable, atom_names=lig.atom_names)


@dataclass
class Grid:
    n: tuple                  # (nx, ny, nz)
    spacing: float
    origin: np.ndarray        # float32 [3], position of node (0,0,0)
    type_names: list          # map order: types, then E, then D
    maps: np.ndarray          # float32 [(n_types+2), nz, ny, nx] (x fastest)

    @property
    def n_types(self):
        return len(self.type_names)

    def type_params(self):
        """float32 [n_types,4] (R, eps, S, V) and int32 roles, in map order."""
        tp = np.array([TYPE_TABLE[t][:4] for t in self.type_names], dtype=np.float32)
        roles = np.array([TYPE_TABLE[t][4] for t in self.type_names], dtype=np.int32)
        return tp, roles


def _pseudo_receptor(rng, lo, hi, pocket_r):
    """Random receptor atoms at ~0.1 atoms/Å^3 filling [lo,hi]^3 minus a carved pocket."""
    vol = float(np.prod(hi - lo))
    n = int(0.1 * vol)
    pts = rng.uniform(lo, hi, size=(n, 3))
    keep = np.linalg.norm(pts, axis=1) > pocket_r
    # random carving so the pocket is not spherical
    for _ in range(6):
        c = _unit(rng.normal(size=3)) * pocket_r * rng.uniform(0.7, 1.1)
        r = pocket_r * rng.uniform(0.35, 0.6)
        keep &= np.linalg.norm(pts - c, axis=1) > r
    pts = pts[keep]
    rtype = rng.choice(4, size=len(pts), p=[0.60, 0.15, 0.20, 0.05])  # C N OA HD
    q = np.where(rng.random(len(pts)) < 0.5, 0.3, -0.3)
    q = q - q.mean()
    return pts, rtype, q


RECEPTOR_TYPES = ["C", "N", "OA", "HD"]


def make_grid(n: int, spacing: float, type_names, seed: int, cutoff: float = 8.0) -> Grid:
    """Receptor maps on an n^3 grid centred on 0 (SURVEY.md §8(d) receptor recipe).

    Type map   M_t(x) = sum_r Morse_{t,r}(d) + (S_t V_r + S_r V_t) exp(-d^2/2σ^2)
    Elec map   M_E(x) = sum_r 332.06363 q_r / (4 max(d,0.5)^2)
    Desolv map M_D(x) = 0.01097 sum_r V_r exp(-d^2/2σ^2)
    within `cutoff`, σ = 3.6 Å; M_t capped at +1e5 as AutoGrid does.
    The Morse shape (not the ligand's 12-6 form) keeps this receptor recipe
    separate from the ligand scoring arithmetic.
    """
    import torch
    rng = np.random.default_rng(seed)
    L = (n - 1) * spacing
    origin = np.full(3, -L / 2.0)
    margin = 4.0
    pts, rtype, rq = _pseudo_receptor(rng, origin - margin, origin + L + margin, 0.3 * L + 2.0)
    sigma2 = 2.0 * 3.6 ** 2
    a_morse = 3.0
    g = np.arange(n) * spacing + origin[0]
    # node coordinates, x fastest
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
    nodes = np.stack([X.ravel(), Y.ravel(), Z.ravel()], axis=1)
    nt = len(type_names)
    out = np.zeros((nt + 2, nodes.shape[0]), dtype=np.float64)
    # cell lists
    cell = cutoff
    cidx = np.floor((pts - (origin - margin)) / cell).astype(np.int64)
    ncell = cidx.max(axis=0) + 1
    key = (cidx[:, 2] * ncell[1] + cidx[:, 1]) * ncell[0] + cidx[:, 0]
    order = np.argsort(key, kind="stable")
    key_s = key[order]
    starts = np.searchsorted(key_s, np.arange(ncell.prod()), side="left")
    ends = np.searchsorted(key_s, np.arange(ncell.prod()), side="right")
    ncid = np.floor((nodes - (origin - margin)) / cell).astype(np.int64)
    nkey = (ncid[:, 2] * ncell[1] + ncid[:, 1]) * ncell[0] + ncid[:, 0]
    rp = np.array([TYPE_TABLE[t] for t in RECEPTOR_TYPES])
    Rr, er, Sr, Vr, rolr = (rp[rtype, i] for i in range(5))
    tt = np.array([TYPE_TABLE[t] for t in type_names])
    torch.set_num_threads(max(1, os.cpu_count() or 1))
    for ck in np.unique(nkey):
        sel = np.nonzero(nkey == ck)[0]
        cz, rem = divmod(ck, ncell[0] * ncell[1])
        cy, cx = divmod(rem, ncell[0])
        cand = []
        for dz in (-1, 0, 1):
            for dy in (-1, 0, 1):
                for dx in (-1, 0, 1):
                    x, y, z = cx + dx, cy + dy, cz + dz
                    if 0 <= x < ncell[0] and 0 <= y < ncell[1] and 0 <= z < ncell[2]:
                        k = (z * ncell[1] + y) * ncell[0] + x
                        cand.append(order[starts[k]:ends[k]])
        cand = np.concatenate(cand)
        if cand.size == 0:
            continue
        P = torch.from_numpy(nodes[sel])
        A = torch.from_numpy(pts[cand])
        d = torch.cdist(P, A)                      # [nsel, ncand]
        within = (d < cutoff).double()
        gauss = torch.exp(-(d * d) / sigma2) * within
        Vr_c = torch.from_numpy(Vr[cand])
        Sr_c = torch.from_numpy(Sr[cand])
        # elec and desolvation maps
        qr = torch.from_numpy(rq[cand])
        dm = torch.clamp(d, min=0.5)
        out[nt, sel] = ((332.06363 * qr / (4.0 * dm * dm)) * within).sum(1).numpy()
        out[nt + 1, sel] = (0.01097 * (gauss * Vr_c).sum(1)).numpy()
        Rr_c = torch.from_numpy(Rr[cand]); er_c = torch.from_numpy(er[cand])
        rol_c = torch.from_numpy(rolr[cand])
        for ti in range(nt):
            Rt, et, St, Vt, rolt = tt[ti]
            hb = ((rol_c == 1) & bool(rolt == 2)) | ((rol_c == 2) & bool(rolt == 1))
            r0 = torch.where(hb, torch.full_like(Rr_c, 1.9), 0.5 * (Rt + Rr_c))
            eps = torch.where(hb, torch.full_like(er_c, 5.0 * 0.2), torch.sqrt(et * er_c))
            ex = torch.exp(-a_morse * (d - r0[None, :]))
            morse = eps[None, :] * ((1.0 - ex) ** 2 - 1.0)
            desolv = (St * Vr_c + Sr_c * Vt)[None, :] * gauss
            v = ((morse + desolv) * within).sum(1)
            out[ti, sel] = torch.clamp(v, max=1e5).numpy()
    maps = out.astype(np.float32).reshape(nt + 2, n, n, n)
    return Grid(n=(n, n, n), spacing=float(spacing), origin=origin.astype(np.float32),
                type_names=list(type_names), maps=maps)


def _cache_dir():
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "build", "inputs")
    os.makedirs(d, exist_ok=True)
    return d


def grid_for_ligand(cfg: Config, type_names) -> Grid:
    """Cached make_grid for a config (cache under build/inputs, git-ignored)."""
    key = f"grid_{cfg.grid_n}_{cfg.spacing}_{cfg.grid_seed}_{'-'.join(type_names)}.npz"
    path = os.path.join(_cache_dir(), key)
    if os.path.exists(path):
        z = np.load(path)
        return Grid(n=tuple(int(v) for v in z["n"]), spacing=float(z["spacing"]),
                    origin=z["origin"], type_names=list(type_names), maps=z["maps"])
    g = make_grid(cfg.grid_n, cfg.spacing, type_names, cfg.grid_seed)
    tmp = path + f".{os.getpid()}.tmp.npz"
    np.savez(tmp, n=np.array(g.n), spacing=np.float64(g.spacing), origin=g.origin, maps=g.maps)
    os.replace(tmp, path)
    return g


def _map_types(lig_types, n_maps):
    """Grid type list: the ligand's types padded (S:83 order) to n_maps-2 types."""
    ts = [t for t in TYPE_NAMES if t in set(lig_types)]
    for t in TYPE_NAMES:
        if len(ts) >= n_maps - 2:
            break
        if t not in ts:
            ts.append(t)
    return [t for t in TYPE_NAMES if t in ts]


def config_inputs(name: str):
    """(Config, Ligand, Grid) for a graded config; the ligand is typed in grid map order."""
    cfg = CONFIGS[name]
    if name == "hts":
        tnames = list(TYPE_NAMES)
        return cfg, None, grid_for_ligand(cfg, tnames)
    lig = make_ligand(cfg.n_atoms, cfg.n_tors, cfg.lig_seed)
    tnames = _map_types(lig.atom_names, cfg.n_maps)
    lig = retype(lig, tnames)
    return cfg, lig, grid_for_ligand(cfg, tnames)


def hts_ligands(n_ligs: int, seed: int = 5):
    """configs[4]: N ~ U{10..70}, T = clip(floor(N/5) + U{-1,0,1}, 0, 15); all 8 types."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n_ligs):
        n = int(rng.integers(10, 71))
        t = int(np.clip(n // 5 + int(rng.integers(-1, 2)), 0, 15))
        out.append(make_ligand(n, t, (seed << 32) | i, type_names=list(TYPE_NAMES)))
    return out


# ---------------------------------------------------------------------------
# Special grids used by the pins (SURVEY.md §8(c) "Special grids for pins").
# ---------------------------------------------------------------------------
def multilinear_grid(n, spacing, origin, coef, type_names=("C",)):
    """M(x,y,z) = a + b x + c y + d z + e xy + f yz + g xz + h xyz at the nodes (grid units)."""
    a, b, c, d, e, f, g, h = coef
    i = np.arange(n, dtype=np.float64)
    Z, Y, X = np.meshgrid(i, i, i, indexing="ij")
    M = a + b * X + c * Y + d * Z + e * X * Y + f * Y * Z + g * X * Z + h * X * Y * Z
    nt = len(type_names)
    maps = np.zeros((nt + 2, n, n, n), dtype=np.float32)
    for t in range(nt):
        maps[t] = M.astype(np.float32)
    return Grid(n=(n, n, n), spacing=float(spacing), origin=np.asarray(origin, np.float32),
                type_names=list(type_names), maps=maps)


def planted_grid(n, spacing, node, a=1.0, type_names=("C",)):
    """M = a·|x - x*|^2 with a unique node minimum x* (S:503 planted minimum)."""
    L = (n - 1) * spacing
    origin = np.full(3, -L / 2.0, dtype=np.float32)
    g = np.arange(n) * spacing + origin[0]
    Z, Y, X = np.meshgrid(g, g, g, indexing="ij")
    xs = origin + np.asarray(node) * spacing
    M = a * ((X - xs[0]) ** 2 + (Y - xs[1]) ** 2 + (Z - xs[2]) ** 2)
    nt = len(type_names)
    maps = np.zeros((nt + 2, n, n, n), dtype=np.float32)
    for t in range(nt):
        maps[t] = M.astype(np.float32)
    return Grid(n=(n, n, n), spacing=float(spacing), origin=origin, type_names=list(type_names), maps=maps)


def constant_grid(n, spacing, value, type_names=("C",)):
    L = (n - 1) * spacing
    origin = np.full(3, -L / 2.0, dtype=np.float32)
    nt = len(type_names)
    maps = np.full((nt + 2, n, n, n), value, dtype=np.float32)
    return Grid(n=(n, n, n), spacing=float(spacing), origin=origin, type_names=list(type_names), maps=maps)


def random_genotypes(grid: Grid, n_tors: int, n: int, seed: int, frac_out: float = 0.05,
                     shrink: float = 0.35):
    """Seeded genotypes for parity tests: translations mostly near the box centre
    (so most atoms are inside), a fraction outside the box, unwrapped angles."""
    rng = np.random.default_rng(seed)
    L = (np.array(grid.n) - 1) * grid.spacing
    lo = grid.origin.astype(np.float64)
    centre = lo + L / 2
    G = 6 + n_tors
    x = np.empty((n, G), dtype=np.float32)
    t = centre + rng.uniform(-shrink, shrink, size=(n, 3)) * L
    out = rng.random(n) < frac_out
    t[out] = lo + rng.uniform(-0.3, 1.3, size=(int(out.sum()), 3)) * L
    x[:, 0:3] = t
    x[:, 3:6] = rng.uniform(-2 * math.pi, 4 * math.pi, size=(n, 3))
    x[:, 6:] = rng.uniform(-2 * math.pi, 4 * math.pi, size=(n, n_tors))
    return x
