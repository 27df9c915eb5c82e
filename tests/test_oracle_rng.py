"""Pins for the oracle's D2 RNG (NS "counter-based Philox RNG")."""
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "philox4x32_10_kat.txt")


def _kat():
    rows = []
    for line in open(GOLD):
        if line.startswith("#") or not line.strip():
            continue
        v = [int(x, 16) for x in line.split()]
        rows.append((v[0:4], v[4:6], v[6:10]))
    return rows


@pytest.mark.parametrize("ctr,key,out", _kat())
def test_philox_known_answers(orc, ctr, key, out):
    assert list(orc.philox(ctr, key)) == out


def test_u01_below_edges(orc):
    assert orc.u01(0) == 0.0
    assert orc.u01(0xFFFFFFFF) == 1.0 - 2.0 ** -24
    assert orc.u01(0x80000000) == 0.5
    for n in (1, 2, 7, 150, 1 << 20):
        assert orc.below(0xFFFFFFFF, n) == n - 1
        assert orc.below(0, n) == 0
    # below is floor(w*n/2^32): exact on powers of two
    assert orc.below(0x40000000, 4) == 1
    assert orc.below(0x3FFFFFFF, 4) == 0


def test_word_layout(orc):
    """word m = lane (m & 3) of the call with block m >> 2 (D2 word map)."""
    seed, lig = 42, 3
    s = (seed + lig * 0x9E3779B97F4A7C15) % 2**64
    key = [s & 0xFFFFFFFF, s >> 32]
    for purpose, slot, gen, run in [(0, 5, 0, 1), (1, 149, 7, 19), (3, 12, 300, 99)]:
        for m in range(0, 40, 3):
            blk = orc.philox([m >> 2, (purpose << 24) | slot, gen, run], key)
            assert orc.word(seed, lig, purpose, slot, gen, run, m) == int(blk[m & 3])


def test_u01_uniformity(orc):
    """Chi-square of 20k u01 draws over 20 bins (distributional sanity)."""
    w = [orc.word(7, 0, 1, k, 1, 0, 0) for k in range(20000)]
    u = np.array([orc.u01(x) for x in w])
    h, _ = np.histogram(u, bins=20, range=(0, 1))
    chi2 = ((h - 1000.0) ** 2 / 1000.0).sum()
    assert chi2 < 50.0          # 19 dof, p ~ 1e-4 cut
