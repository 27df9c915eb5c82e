"""Golden hand traces pinning the oracle's D8-D10 search steps word by word (VERDICT r1:
the permutation / bowl / rate pins alone let a shifted word index, swapped bias
coefficients or a wrong s_d update pass).  Each trace in tests/golden/ is worked by hand
from explicit Philox words (the words themselves are tied to the KAT-pinned Philox here).
"""
import math
import os

import numpy as np
import pytest

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _rows(name):
    rows, kv = [], {}
    for line in open(os.path.join(GOLD, name)):
        line = line.strip()
        if not line or line.startswith("#"):
            continue
        f = line.split()
        if f[0][0].isalpha():
            kv[f[0]] = f[1:]
        else:
            rows.append([float(v) for v in f])
    return rows, kv


def test_solis_wets_bowl_hand_trace(orc):
    rows, kv = _rows("sw_bowl_trace.txt")
    words = [int(w, 16) for w in kv["words"]]
    assert [orc.word(2022, 0, 3, 7, 2, 3, m) for m in range(len(words))] == words
    pp = orc.params(ls_max_iters=6, sw_cons_succ=2, sw_cons_fail=1)
    x, E, ev, to, tr, tE = orc.solis_wets_traced(None, pp, 2022, 0, 3, 2, 7, np.array([5.0]), 25.0,
                                                 bowl=np.array([1.0]))
    n_eval = 0
    for r in rows:
        it, rho, d, c1, E1, c2, E2, o, xr, br, Ex = r
        it, o = int(it), int(o)
        assert to[it] == o and tr[it] == rho, it
        assert tE[it, 1] == pytest.approx(E1, rel=1e-14), it
        if math.isnan(E2):
            assert math.isnan(tE[it, 2]), it
        else:
            assert tE[it, 2] == pytest.approx(E2, rel=1e-14), it
        n_eval += 1 if math.isnan(E2) else 2
    xr, Ex = rows[-1][8], rows[-1][10]
    assert x[0] == pytest.approx(xr, rel=1e-14) and E == pytest.approx(Ex, rel=1e-14)
    assert ev == n_eval == 10


def test_adadelta_bowl_hand_trace(orc):
    rows, _ = _rows("adadelta_bowl_trace.txt")
    pp = orc.params()
    x, E, ev, tx, tE, tg = orc.adadelta_traced(None, pp, 3, np.array([1.0, 1.0]), 1e30, bowl=np.array([1.0, 10.0]))
    for r in rows:
        it = int(r[0])
        assert tx[it] == pytest.approx(r[1:3], rel=1e-14), it
        assert tE[it] == pytest.approx(r[3], rel=1e-14), it
    assert x == pytest.approx(rows[2][1:3], rel=1e-14) and E == pytest.approx(rows[2][3], rel=1e-14)
    assert ev == 3


def test_ls_pick_hand_trace(orc):
    _, kv = _rows("ga_ls_pick_trace.txt")
    words = [int(w, 16) for w in kv["pick_words"]]
    assert [orc.word(2022, 0, 2, 0, 4, 1, m) for m in range(3)] == words
    assert list(orc.ls_pick(2022, 0, 1, 4, 10, 3)) == [int(v) for v in kv["pick_perm"]]


def test_ga_slot_word_map_hand_trace(orc):
    _, kv = _rows("ga_ls_pick_trace.txt")
    words = [int(w, 16) for w in kv["ga_words"]]
    assert [orc.word(2022, 0, 1, 2, 5, 0, m) for m in range(len(words))] == words
    old = np.array([[10.0 + i, 20.0 + i, 30.0 + i, 40.0 + i] for i in range(4)])
    E = np.array([3.0, -1.0, 2.0, -1.0])
    pp = orc.params(p_tour=0.6, p_cross=0.8, p_mut=0.5)
    child, dbg = orc.ga_slot(pp, 2022, 0, 0, 5, 2, old, E)
    A, B, cross, c1, c2 = (int(v) for v in kv["ga_debug"][:5])
    assert list(dbg[:5]) == [A, B, cross, c1, c2]
    assert dbg[5] == (1 << 0) | (1 << 2)                  # genes 0 and 2 mutated
    assert child == pytest.approx([float(v) for v in kv["ga_child"]], rel=1e-15)


def test_generation0_hand_trace(orc):
    from gen.synth import constant_grid
    _, kv = _rows("ga_ls_pick_trace.txt")
    words = [int(w, 16) for w in kv["init_words"]]
    assert [orc.word(2022, 0, 0, 1, 0, 0, m) for m in range(6)] == words
    grid = constant_grid(11, 1.0, 0.0)
    assert np.allclose(grid.origin, -5.0)
    P = orc.Problem(grid, types=np.zeros(1, np.int32), charges=np.zeros(1, np.float32),
                    xyz=np.zeros((1, 3), np.float32), bonds=np.zeros((0, 2), np.int32),
                    rotatable=np.zeros(0, np.uint8))
    g, E = orc.init_population(P, 3, 2022, run=0)
    assert g[1] == pytest.approx([float(v) for v in kv["init_genes"]], rel=1e-15)
    assert (E == 0.0).all()                               # constant zero maps, no pairs
