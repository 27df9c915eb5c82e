"""SPEC-style verbatim torsions and pairs (reading D1.7; SURVEY.md §8(b) `dock_ligand.n_tors /
tors_* / n_pairs / pairs`).  The oracle's brute-force validation
(or_topology_verbatim) and the library's (prep.cpp verbatim_topology, through the
host-only dock_topology) are independent; both must accept and reject the same hand cases,
and an accepted topology must come back unchanged.  The oracle's D7 gradient on a
non-D1 verbatim topology is pinned by central differences."""
import numpy as np
import pytest

import oracle
from gen import config_inputs, random_genotypes
from gen.synth import TYPE_NAMES


@pytest.fixture(scope="module")
def dock():
    from paper_2203_02096_b200._build import build
    build()
    import paper_2203_02096_b200 as d
    return d


def chain(n):
    """A zig-zag chain 0-1-...-(n-1) (coordinates only matter for non-zero axes)."""
    xyz = np.array([[1.4 * i, 0.5 * (i % 2), 0.0] for i in range(n)], np.float32)
    return dict(types=np.zeros(n, np.int32), charges=np.zeros(n, np.float32), xyz=xyz)


def both(dock, lig, axis, moved, pairs):
    """(oracle verdict, ABI verdict) as (ok, topology) pairs."""
    n = len(lig["types"])
    try:
        o = oracle.topology_verbatim(n, axis, moved, pairs)
    except ValueError:
        o = None
    tp = np.array([[4.0, 0.15, -0.001, 30.0]] * len(TYPE_NAMES), np.float32)
    roles = np.zeros(len(TYPE_NAMES), np.int32)
    try:
        a = dock.topology(lig["types"], lig["charges"], lig["xyz"], None, None, tp, roles,
                          tors=(np.asarray(axis).reshape(-1, 2), moved), pairs=np.asarray(pairs).reshape(-1, 2))
    except dock.DockError as e:
        assert e.code == dock.DOCK_E_INPUT
        a = None
    return o, a


# chain 0-1-2-3-4-5-6-7: torsion about 2->3 moves {4..7}; nested torsion about 4->5 moves {6, 7}
AX = [[2, 3], [4, 5]]
MV = [[4, 5, 6, 7], [6, 7]]
PR = [[0, 4], [0, 5], [7, 1]]

CASES = [
    ("valid chain", AX, MV, PR, True),
    ("no torsions, no pairs", np.zeros((0, 2)), [], np.zeros((0, 2)), True),
    ("disjoint sets", [[2, 3], [2, 1]], [[4, 5, 6, 7], [0]], PR, True),
    ("empty moved set", [[2, 3], [5, 6]], [[4, 5, 6, 7], []], PR, True),
    ("overlapping sets", [[2, 3], [5, 1]], [[4, 5, 6], [6, 7]], PR, False),
    ("child before parent", [[4, 5], [2, 3]], [[6, 7], [4, 5, 6, 7]], PR, False),
    ("later torsion moves an earlier axis", [[2, 3], [0, 1]], [[4, 5, 6, 7], [2, 3, 4, 5, 6, 7]], PR, False),
    ("nested axis not carried", [[2, 3], [1, 5]], [[4, 5, 6, 7], [6, 7]], PR, False),
    ("moved contains its axis", [[2, 3], [4, 5]], [[3, 4, 5, 6, 7], [6, 7]], PR, False),
    ("duplicate moved atom", [[2, 3]], [[4, 4, 5]], PR, False),
    ("axis atoms equal", [[2, 2]], [[4, 5]], PR, False),
    ("axis out of range", [[2, 8]], [[4, 5]], PR, False),
    ("moved out of range", [[2, 3]], [[4, 9]], PR, False),
    ("self pair", AX, MV, [[0, 4], [3, 3]], False),
    ("duplicate pair (reversed)", AX, MV, [[0, 4], [4, 0]], False),
    ("pair out of range", AX, MV, [[0, 8]], False),
]


@pytest.mark.parametrize("name,axis,moved,pairs,ok", CASES, ids=[c[0] for c in CASES])
def test_verbatim_validation_hand_cases(dock, name, axis, moved, pairs, ok):
    lig = chain(8)
    o, a = both(dock, lig, axis, moved, pairs)
    assert (o is not None) == ok and (a is not None) == ok, (name, o, a)
    if ok:
        T = np.asarray(axis).reshape(-1, 2).shape[0]
        assert np.array_equal(o["tor_a"], np.asarray(axis, np.int32).reshape(-1, 2)[:, 0])
        ax, mv, pr = a
        assert np.array_equal(ax, np.asarray(axis, np.int32).reshape(-1, 2))     # torsion order kept
        for k in range(T):
            assert set(np.nonzero(mv[k])[0]) == set(moved[k]) == set(np.nonzero(o["moved"][k])[0])
        want = np.sort(np.asarray(pairs, np.int32).reshape(-1, 2), axis=1)      # i < j, list order
        assert np.array_equal(pr, want) and np.array_equal(o["pairs"], want)


def test_rotatable_flags_rejected_with_verbatim_torsions(dock):
    lig = chain(8)
    bonds = np.array([[i, i + 1] for i in range(7)], np.int32)
    rot = np.zeros(7, np.uint8); rot[2] = 1
    tp = np.array([[4.0, 0.15, -0.001, 30.0]] * len(TYPE_NAMES), np.float32)
    with pytest.raises(dock.DockError) as e:
        dock.topology(lig["types"], lig["charges"], lig["xyz"], bonds, rot, tp, np.zeros(len(TYPE_NAMES), np.int32),
                      tors=(np.array(AX), MV), pairs=np.array(PR))
    assert e.value.code == dock.DOCK_E_INPUT


@pytest.mark.parametrize("name", ["1stp", "3ce3", "7cpa"])
def test_derived_topology_round_trips_verbatim(dock, name):
    """The D1-derived topology, fed back verbatim, is accepted by both sides unchanged."""
    cfg, lig, grid = config_inputs(name)
    tp, roles = grid.type_params()
    ax, mv, pr = dock.topology(lig.types, lig.charges, lig.xyz, lig.bonds, lig.rotatable, tp, roles)
    moved = [list(np.nonzero(mv[k])[0]) for k in range(ax.shape[0])]
    ax2, mv2, pr2 = dock.topology(lig.types, lig.charges, lig.xyz, None, None, tp, roles, tors=(ax, moved), pairs=pr)
    assert np.array_equal(ax, ax2) and np.array_equal(mv, mv2) and np.array_equal(pr, pr2)
    o = oracle.topology_verbatim(len(lig.types), ax, moved, pr)
    ref = oracle.topology(len(lig.types), lig.bonds, lig.rotatable)
    for k in ("tor_a", "tor_b", "moved", "pairs"):
        assert np.array_equal(o[k], ref[k]), k


def spec_style(lig, topo, drop=(1,), pair_keep=0.7, seed=3):
    """A verbatim topology that D1 would not produce: a subset of the derived torsions (the
    rest frozen) and a random subset of the pairs, listed in shuffled order."""
    rng = np.random.default_rng(seed)
    keep = [k for k in range(topo["T"]) if k not in drop]
    axis = np.stack([topo["tor_a"][keep], topo["tor_b"][keep]], 1)
    moved = [list(np.nonzero(topo["moved"][k])[0]) for k in keep]
    pr = topo["pairs"][rng.random(topo["pairs"].shape[0]) < pair_keep]
    pr = pr[rng.permutation(pr.shape[0])]
    pr[::3] = pr[::3, ::-1]                                   # some pairs listed (j, i)
    return axis, moved, pr


def test_oracle_gradient_on_verbatim_topology(orc):
    """D7 on a non-D1 verbatim topology (rules (d), (e) keep the world axes right): the
    analytic gradient equals central differences of the oracle's energy."""
    cfg, lig, grid = config_inputs("3ce3")
    ref = oracle.topology(len(lig.types), lig.bonds, lig.rotatable)
    axis, moved, pr = spec_style(lig, ref, drop=(0, 3))
    topo = oracle.topology_verbatim(len(lig.types), axis, moved, pr)
    P = oracle.Problem(grid, lig, topo=topo)
    assert P.T == ref["T"] - 2 and P.P == pr.shape[0]
    X = random_genotypes(grid, P.T, 30, seed=5, frac_out=0.0, shrink=0.2).astype(np.float64)
    checked = 0
    for x in X:
        r = P.energy(x)
        fm, cm = P.margins(r["xyz"])
        if fm < 1e-3 or cm < 1e-3:
            continue
        fd = np.zeros_like(x)
        for j in range(x.shape[0]):
            xp = x.copy(); xp[j] += 1e-6
            xm = x.copy(); xm[j] -= 1e-6
            fd[j] = (P.energy(xp, grad=False)["E"] - P.energy(xm, grad=False)["E"]) / 2e-6
        scale = max(np.abs(r["grad"]).max(), 1.0)
        assert np.abs(fd - r["grad"]).max() <= 1e-5 * scale + 1e-9 * abs(r["E"]) / 1e-6
        checked += 1
    assert checked >= 20
