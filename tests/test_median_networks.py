"""CPU pins of the median identities the fused kernel's networks rely on
(kernel_fused.cuh med3 / med9 / med5; DESIGN.md 6.1 step 4 and 5).

Hybrid median, PAPER.md:76 (Sec. 3.4): med3(median of the '+' group, median of
the 'x' group, centre).  The kernel evaluates
  med3(a, b, c)   = a ^ b ^ c ^ min3 ^ max3        (the element that is neither)
  med9(v0..v8)    = med3(max of the three triple minima, med3 of the triple
                         medians, min of the three triple maxima)
  med5(a,b,c,d,e) = med3(max(min(a,b), min(c,d)), min(max(a,b), max(c,d)), e)
The XOR form is not a min/max network, so the 0-1 principle does not cover it:
these tests enumerate multi-valued inputs exhaustively (4^9 for med9, 5^5 for
med5, 6^3 for med3), ties included, against sorting.
"""
import itertools

import numpy as np


def med3(a, b, c):
    lo = np.minimum(np.minimum(a, b), c)
    hi = np.maximum(np.maximum(a, b), c)
    return a ^ b ^ c ^ lo ^ hi


def med9(v):
    tri = [v[0:3], v[3:6], v[6:9]]
    lows = [np.minimum(np.minimum(t[0], t[1]), t[2]) for t in tri]
    highs = [np.maximum(np.maximum(t[0], t[1]), t[2]) for t in tri]
    mids = [med3(*t) for t in tri]
    L = np.maximum(np.maximum(lows[0], lows[1]), lows[2])
    Hh = np.minimum(np.minimum(highs[0], highs[1]), highs[2])
    return med3(L, med3(*mids), Hh)


def med5(a, b, c, d, e):
    return med3(np.maximum(np.minimum(a, b), np.minimum(c, d)), np.minimum(np.maximum(a, b), np.maximum(c, d)), e)


def _all(values, n):
    g = np.array(list(itertools.product(values, repeat=n)), dtype=np.uint32)
    return [g[:, i] for i in range(n)]


def test_med3_exhaustive():
    v = _all([0, 1, 2, 3, 0x8000, 0xFFFF], 3)
    assert np.array_equal(med3(*v), np.sort(np.stack(v), axis=0)[1])


def test_med9_exhaustive_4_values():
    v = _all([0, 1, 2, 3], 9)
    assert np.array_equal(med9(v), np.sort(np.stack(v), axis=0)[4])


def test_med9_random_wide():
    rng = np.random.default_rng(9)
    v = [rng.integers(0, 65536, 200000, dtype=np.uint32) for _ in range(9)]
    assert np.array_equal(med9(v), np.sort(np.stack(v), axis=0)[4])


def test_med5_exhaustive_5_values():
    v = _all([0, 1, 2, 3, 4], 5)
    assert np.array_equal(med5(*v), np.sort(np.stack(v), axis=0)[2])


def test_packed_pairs_are_independent():
    """The kernel runs the networks on two u16 values per 32-bit word (min/max
    .u16x2, XOR bitwise): the halves never interact."""
    rng = np.random.default_rng(10)
    lo = [rng.integers(0, 65536, 50000, dtype=np.uint32) for _ in range(9)]
    hi = [rng.integers(0, 65536, 50000, dtype=np.uint32) for _ in range(9)]

    def vmin(a, b):
        return np.minimum(a & 0xFFFF, b & 0xFFFF) | (np.minimum(a >> 16, b >> 16) << 16)

    def vmax(a, b):
        return np.maximum(a & 0xFFFF, b & 0xFFFF) | (np.maximum(a >> 16, b >> 16) << 16)

    def pmed3(a, b, c):
        return a ^ b ^ c ^ vmin(vmin(a, b), c) ^ vmax(vmax(a, b), c)

    def pmed9(v):
        tri = [v[0:3], v[3:6], v[6:9]]
        L = vmax(vmax(*[vmin(vmin(*t[:2]), t[2]) for t in tri][:2]), vmin(vmin(*tri[2][:2]), tri[2][2]))
        Hh = vmin(vmin(*[vmax(vmax(*t[:2]), t[2]) for t in tri][:2]), vmax(vmax(*tri[2][:2]), tri[2][2]))
        return pmed3(L, pmed3(*[pmed3(*t) for t in tri]), Hh)

    packed = [a | (b << 16) for a, b in zip(lo, hi)]
    got = pmed9(packed)
    assert np.array_equal(got & 0xFFFF, np.sort(np.stack(lo), axis=0)[4])
    assert np.array_equal(got >> 16, np.sort(np.stack(hi), axis=0)[4])
