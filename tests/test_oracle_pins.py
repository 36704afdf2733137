"""Pins of the CPU oracle against what the paper and mathematics fix.

Every test here checks the oracle (oracle/lfe_oracle.c) against something other
than itself: closed forms, a different computational route (finite-difference
Laplacian of the Gaussian, scipy.ndimage, statistics.stdev/median), worked
examples (SPEC.md, SURVEY.md appendices), invariants (dihedral, negation,
linearity) and brute force on tiny inputs.  CPU only.
"""
import itertools
import math
import os
import statistics

import numpy as np
import pytest
import scipy.ndimage as ndi

import oracle as O
from paper_1304_3992_b200 import scenes

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def _golden_rows(name):
    rows = []
    with open(os.path.join(GOLDEN, name)) as f:
        for line in f:
            line = line.strip()
            if line and not line.startswith("#"):
                rows.append([float(v) for v in line.split()])
    return rows


# ----------------------------------------------------------------- Eq. 1 ----
@pytest.mark.parametrize("sigma", [0.5, 0.8, 1.0, 2.0, 5.0, 20.0])
def test_eq1_is_laplacian_of_normalised_gaussian(sigma):
    """Eq. 1 is the Laplacian of G = exp(-r^2/2s^2)/(2 pi s^2).

    Route independent of the formula: a 5-point finite-difference Laplacian of
    the Gaussian itself (step h, O(h^2) error).
    """
    def G(x, y):
        return math.exp(-(x * x + y * y) / (2 * sigma * sigma)) / (2 * math.pi * sigma * sigma)

    h = 1e-3 * sigma
    raw = O.log_raw(sigma, 5)
    for y in range(-2, 3):
        for x in range(-2, 3):
            fd = (G(x + h, y) + G(x - h, y) + G(x, y + h) + G(x, y - h) - 4 * G(x, y)) / (h * h)
            scale = 1.0 / (math.pi * sigma ** 4)
            assert abs(raw[y + 2, x + 2] - fd) <= 1e-5 * scale, (x, y, raw[y + 2, x + 2], fd)


def test_eq1_centre_closed_form():
    """sigma = 1 centre = -1/pi."""
    assert O.log_raw(1.0, 5)[2, 2] == pytest.approx(-1.0 / math.pi, rel=1e-15)
    for s in (0.5, 3.0, 20.0):
        assert O.log_raw(s, 3)[1, 1] == pytest.approx(-1.0 / (math.pi * s ** 4), rel=1e-14)


def test_eq1_zero_ring():
    """Eq. 1 vanishes where x^2 + y^2 = 2 sigma^2."""
    assert abs(O.log_raw(1.0, 5)[3, 3]) < 1e-17          # (1,1), sigma = 1
    raw = O.log_raw(math.sqrt(0.5), 5)                    # (1,0) ring, sigma^2 = 0.5
    for (y, x) in [(1, 2), (3, 2), (2, 1), (2, 3)]:
        assert abs(raw[y, x]) < 1e-15 * abs(raw[2, 2])  # sqrt(0.5)^2 != 0.5 exactly


@pytest.mark.parametrize("sigma,n", [(0.5, 5), (20.0, 5), (1.3, 3), (2.0, 7), (0.7, 7)])
def test_dc_mask_zero_sum_and_8fold_symmetry(sigma, n):
    L = O.log_dc(sigma, n)
    assert abs(L.sum()) < 1e-12 * np.abs(L).sum()
    for T in (L.T, L[::-1, :], L[:, ::-1], L[::-1, ::-1]):
        np.testing.assert_array_equal(L, T)


def test_raw_sigma20_has_no_sign_change_dc_is_mandatory():
    """Reading R2: the raw 5x5 sigma=20 mask is strictly negative, so without DC
    correction it cannot produce a zero crossing."""
    raw = O.log_raw(20.0, 5)
    assert (raw < 0).all()


def test_dc_large_sigma_limit():
    """For sigma >> window, Eq. 1 ~ c0 + c1 (x^2+y^2) (Taylor), so the DC-corrected
    5x5 mask -> (x^2 + y^2 - 4)/4 after dividing by |centre|."""
    L = O.log_dc(20.0, 5)
    L = L / abs(L[2, 2])
    y, x = np.mgrid[-2:3, -2:3]
    np.testing.assert_allclose(L, (x * x + y * y - 4) / 4.0, atol=0.005)


# ------------------------------------------------------- integer masks ----
@pytest.mark.parametrize("row", _golden_rows("masks_A2.txt"))
def test_integer_masks_match_survey_table(row):
    sigma, b, F, sabs, *orb = row
    q, Fo = O.mask_int(sigma, 5, int(b))
    assert Fo == int(F)
    assert int(np.abs(q).sum()) == int(sabs)
    got = [q[2, 2], q[2, 3], q[2, 4], q[3, 3], q[3, 4], q[4, 4]]
    assert [int(v) for v in got] == [int(v) for v in orb]


@pytest.mark.parametrize("sigma", [0.5, 0.9, 1.7, 4.0, 20.0])
@pytest.mark.parametrize("n", [3, 5, 7])
@pytest.mark.parametrize("b", [1, 8, 10, 12, 16])
def test_integer_mask_properties(sigma, n, b):
    """Zero sum, 8-fold symmetry, |r| < 2^24 bound, F maximal (reading R3)."""
    q, F = O.mask_int(sigma, n, b)
    M = (1 << b) - 1
    assert int(q.sum()) == 0
    for T in (q.T, q[::-1, :], q[:, ::-1]):
        np.testing.assert_array_equal(q, T)
    assert M * int(np.abs(q).sum()) < (1 << 24)
    if F < 16:  # F + 1 must violate the bound
        L = O.log_dc(sigma, n)
        c = abs(L[n // 2, n // 2])
        q1 = np.array([[math.copysign(math.floor(abs(v / c * 2 ** (F + 1)) + 0.5), v)
                        for v in row] for row in L])
        q1[n // 2, n // 2] = 0
        q1[n // 2, n // 2] = -q1.sum()
        assert M * np.abs(q1).sum() >= (1 << 24)


# ------------------------------------------------------------ LoG stage ----
def test_log_constant_image_is_zero():
    for s, b in [(0.5, 8), (20, 10), (1.0, 12)]:
        q, _ = O.mask_int(s, 5, b)
        I = np.full((9, 13), (1 << b) - 1, np.uint16)
        assert not O.log_response(I, q).any()


def test_log_matches_scipy_correlate_nearest():
    """Special case that reduces to a library routine: scipy.ndimage.correlate
    with mode='nearest' is exactly replicate-padded mask application."""
    rng = np.random.default_rng(0)
    for s, n, b in [(0.5, 5, 8), (20, 5, 10), (1.2, 3, 12), (2.0, 7, 8)]:
        q, _ = O.mask_int(s, n, b)
        I = rng.integers(0, 1 << b, (23, 31)).astype(np.uint16)
        ref = ndi.correlate(I.astype(np.int64), q.astype(np.int64), mode="nearest")
        np.testing.assert_array_equal(O.log_response(I, q), ref)


def test_log_kills_linear_ramps_and_quadratic_gives_moment():
    """A symmetric zero-sum mask annihilates a*x + b*y + c; on x^2 it returns the
    constant second moment sum q(d) dx^2 (interior)."""
    q, _ = O.mask_int(0.5, 5, 12)
    y, x = np.mgrid[0:20, 0:20]
    I = (3 * x + 5 * y + 7).astype(np.uint16)
    r = O.log_response(I, q)
    assert not r[2:-2, 2:-2].any()
    I2 = (x * x).astype(np.uint16)
    r2 = O.log_response(I2, q)
    dx = np.arange(-2, 3)[None, :]
    moment = int((q.astype(np.int64) * dx * dx).sum())
    assert (r2[2:-2, 2:-2] == moment).all()


def test_log_linearity():
    rng = np.random.default_rng(1)
    q, _ = O.mask_int(20.0, 5, 8)
    A = rng.integers(0, 100, (15, 17)).astype(np.uint16)
    B = rng.integers(0, 100, (15, 17)).astype(np.uint16)
    np.testing.assert_array_equal(O.log_response(A + 2 * B, q),
                                  O.log_response(A, q) + 2 * O.log_response(B, q))


def test_log_step_profile_matches_survey_A3():
    (row,) = _golden_rows("step_profile_A3.txt")
    q, _ = O.mask_int(0.5, 5, 8)
    I = np.zeros((6, 16), np.uint16)
    I[:, 8:] = 200
    r = O.log_response(I, q)
    for yy in range(6):
        assert [int(v) for v in r[yy, 5:11]] == [int(v) for v in row]


# ------------------------------------------------------------- ZC stage ----
def test_zc_spec_example_row():
    """row [-3, 1]: threshold 2 marks only the 1; 5 marks none."""
    r = np.array([[-3, 1]], np.int64)
    assert O.zero_crossing(r, 2).tolist() == [[0, 1]]
    assert O.zero_crossing(r, 5).tolist() == [[0, 0]]


def test_zc_same_sign_never_marks():
    """'If they all have the same sign ... no zero crossing'."""
    rng = np.random.default_rng(2)
    r = rng.integers(1, 50, (20, 20)).astype(np.int64)
    assert not O.zero_crossing(r).any()
    assert not O.zero_crossing(-r).any()


def _zc_brute(c, nbs, t):
    """Brute force on one cross: the candidate is marked iff some neighbour has
    the strictly opposite sign, no opposite-sign neighbour is smaller in
    magnitude, and the largest opposite pair gap reaches t; a zero candidate
    needs a positive and a negative neighbour spanning >= t."""
    if c == 0:
        pos = [v for v in nbs if v > 0]
        neg = [v for v in nbs if v < 0]
        return int(bool(pos) and bool(neg) and max(nbs) - min(nbs) >= t)
    opp = sorted((abs(v) for v in nbs if v * c < 0))
    if not opp:
        return 0
    return int(abs(c) <= opp[0] and abs(c) + opp[-1] >= t)


def test_zc_exhaustive_crosses():
    """All 5^5 crosses with values in {-3,-1,0,1,3}, thresholds 0..7."""
    vals = [-3, -1, 0, 1, 3]
    pats = list(itertools.product(vals, repeat=5))
    # embed each cross in a 3x3 block whose corners are 0 (corners are not N4)
    blocks = np.zeros((len(pats), 3, 3), np.int64)
    for i, (c, u, d, l, rr) in enumerate(pats):
        blocks[i, 1, 1], blocks[i, 0, 1], blocks[i, 2, 1] = c, u, d
        blocks[i, 1, 0], blocks[i, 1, 2] = l, rr
    # lay the blocks out in a grid separated by... nothing: compute per block so
    # that the 1-row replicate padding of a 3x3 image leaves the centre's N4 intact
    for t in range(0, 8):
        for i, (c, u, d, l, rr) in enumerate(pats):
            Z = O.zero_crossing(blocks[i], t)
            assert Z[1, 1] == _zc_brute(c, [u, d, l, rr], t), (pats[i], t)


def test_zc_step_marks_the_two_straddling_columns():
    """an ideal step is marked on exactly the two columns that
    straddle it, for both masks and 8/10-bit depths (reading R8, ties marked)."""
    for s in (0.5, 20.0):
        for b in (8, 10):
            q, _ = O.mask_int(s, 5, b)
            I = np.zeros((10, 20), np.uint16)
            I[:, 10:] = (1 << b) - 1
            Z = O.zero_crossing(O.log_response(I, q))
            cols = sorted(set(np.nonzero(Z)[1].tolist()))
            assert cols == [9, 10], (s, b, cols)
            assert Z[:, 9].all() and Z[:, 10].all()


def test_zc_threshold_decides_at_the_step_gap():
    """Pins the normalised-threshold conversion t = ceil(thr * 2^F * M) (R9) to
    numbers outside the oracle: the A.3 step (sigma 0.5, 8-bit, A = 200) has one
    opposite-sign pair with gap 2 * 2246600 (golden profile), and A.2 gives F = 15
    for that mask.  The crossing survives exactly up to thr = gap / (2^F * 255):
    a wrong scale, a dropped M or 2^F, or floor instead of ceil flips one case."""
    (row,) = _golden_rows("step_profile_A3.txt")
    gap = int(row[2]) - int(row[3])
    F = next(int(r[2]) for r in _golden_rows("masks_A2.txt") if float(r[0]) == 0.5 and int(r[1]) == 8)
    thr0 = gap / (2.0**F * 255)
    I = np.full((12, 16), 0, np.uint16)
    I[:, 8:] = 200
    def kept(thr):
        p = O.Params(bit_depth=8, sigma=(0.5, 0.5), zc_threshold=(thr, thr), hybrid_median=False, out_mode=1)
        return sorted(set(np.nonzero(O.run(I, p))[1].tolist()))
    assert kept(thr0 * (1 - 1e-12)) == [7, 8]
    assert kept(thr0 * (1 + 1e-9)) == []
    assert kept(0.0) == [7, 8]
    # thresholds far beyond any gap (2^25, R3) reject everything, without overflow
    assert kept(1e30) == [] and kept(1e300) == []
    assert O.zc_threshold_int(1e300, F, 8) >= 2**26


@pytest.mark.parametrize("w", [3, 5, 7])
def test_std_gate_windows_vs_statistics(w):
    """Eq. 2 at every window size of NEXT-4: the gate at the centre
    of a w x w image (no padding reaches it) against statistics.stdev of the
    whole window, for the intensity source and for a binary ZC window."""
    rng = np.random.default_rng(40 + w)
    c = w // 2
    for _ in range(200):
        I = rng.integers(0, 1024, (w, w)).astype(np.uint16)
        Z = np.zeros((w, w), np.uint8)
        Z[c, c] = 1
        T = float(rng.uniform(0, 500))
        keep = O.std_gate(I, Z, w, T)
        assert bool(keep[c, c]) == (statistics.stdev(I.ravel().astype(float)) > T)
        B = (rng.random((w, w)) < rng.uniform(0.05, 0.95)).astype(np.uint8)
        B[c, c] = 1
        Tb = float(rng.uniform(0.05, 0.55))
        keep = O.std_gate(B, B, w, Tb)
        assert bool(keep[c, c]) == (statistics.stdev(B.ravel().astype(float)) > Tb)


def test_zc_ramp_marks_the_middle_column():
    q, _ = O.mask_int(0.5, 5, 8)
    I = np.zeros((8, 17), np.uint16)
    I[:, 8] = 100
    I[:, 9:] = 200
    Z = O.zero_crossing(O.log_response(I, q))
    assert sorted(set(np.nonzero(Z)[1].tolist())) == [8]


@pytest.mark.parametrize("R", [3.0, 5.5, 8.0, 12.3, 15.0, 21.7])
def test_zc_disk_marks_only_boundary_pixels(R):
    """Crossings of a digital disk lie only on pixels 4-adjacent across the
    disk boundary."""
    N = int(2 * R) + 16
    c = N / 2.0
    yy, xx = np.mgrid[0:N, 0:N]
    inside = (xx - c) ** 2 + (yy - c) ** 2 <= R * R
    I = np.where(inside, 200, 30).astype(np.uint16)
    pad = np.pad(inside, 1, mode="edge")
    across = ((pad[1:-1, 1:-1] != pad[:-2, 1:-1]) | (pad[1:-1, 1:-1] != pad[2:, 1:-1])
              | (pad[1:-1, 1:-1] != pad[1:-1, :-2]) | (pad[1:-1, 1:-1] != pad[1:-1, 2:]))
    for s in (0.5, 20.0):
        q, _ = O.mask_int(s, 5, 8)
        Z = O.zero_crossing(O.log_response(I, q)).astype(bool)
        assert Z.any()
        assert not (Z & ~across).any()


_DIHEDRAL = [
    lambda a: a, lambda a: np.rot90(a, 1), lambda a: np.rot90(a, 2), lambda a: np.rot90(a, 3),
    lambda a: a.T, lambda a: a[::-1, :], lambda a: a[:, ::-1], lambda a: np.rot90(a, 1).T,
]


def test_zc_dihedral_and_negation_invariance():
    rng = np.random.default_rng(3)
    for _ in range(20):
        r = rng.integers(-4, 5, (11, 14)).astype(np.int64)
        t = int(rng.integers(0, 5))
        Z = O.zero_crossing(r, t)
        np.testing.assert_array_equal(O.zero_crossing(-r, t), Z)
        for T in _DIHEDRAL:
            np.testing.assert_array_equal(O.zero_crossing(np.ascontiguousarray(T(r)), t), T(Z))


# ------------------------------------------------------------ std stage ----
def test_eq2_worked_example():
    """twenty-four 0s and one 100 -> s = 20 exactly."""
    assert O.sample_std([0] * 24 + [100]) == 20.0


def test_eq2_matches_statistics_stdev():
    rng = np.random.default_rng(4)
    for _ in range(2000):
        a = rng.integers(0, 1024, 25).astype(float)
        assert O.sample_std(a) == pytest.approx(statistics.stdev(a), rel=1e-12, abs=1e-12)
    assert O.sample_std(np.full(9, 7.0)) == 0.0


@pytest.mark.parametrize("T,lo,hi", [(0.2, 2, 23), (0.25, 2, 23), (0.3, 3, 22), (0.35, 4, 21),
                                     (0.4, 5, 20), (0.45, 7, 18), (0.5, 11, 14)])
def test_binary_std_pass_ranges(T, lo, hi):
    """Binary 5x5 window with k ones passes s > T iff lo <= k <= hi,
    checked against statistics.stdev of the window."""
    for k in range(1, 26):
        Z = np.zeros(25, np.uint8)
        Z[12] = 1                                             # the centre is a crossing
        Z[[i for i in range(25) if i != 12][: k - 1]] = 1     # plus k-1 others
        Z = Z.reshape(5, 5)
        keep = O.std_gate(Z, Z, 5, T)
        expect = statistics.stdev(Z.ravel().astype(float)) > T
        assert bool(keep[2, 2]) == expect == (lo <= k <= hi), (k, T)


def test_std_gate_intensity_and_recheck_vs_statistics():
    rng = np.random.default_rng(5)
    for _ in range(300):
        I = rng.integers(0, 1024, (5, 5)).astype(np.uint16)
        Z = np.zeros((5, 5), np.uint8)
        Z[2, 2] = 1
        T = float(rng.uniform(0, 500))
        T3 = float(rng.uniform(0, 500))
        s5 = statistics.stdev(I.ravel().astype(float))
        s3 = statistics.stdev(I[1:4, 1:4].ravel().astype(float))
        keep = O.std_gate(I, Z, 5, T, T3)
        assert bool(keep[2, 2]) == (s5 > T and s3 > T3)
        keep = O.std_gate(I, Z, 5, T)
        assert bool(keep[2, 2]) == (s5 > T)
        assert keep.sum() == keep[2, 2]  # non-crossings are never kept


def test_std_gate_constant_offset_invariance():
    rng = np.random.default_rng(6)
    I = rng.integers(0, 500, (12, 12)).astype(np.uint16)
    Z = (rng.random((12, 12)) < 0.5).astype(np.uint8)
    np.testing.assert_array_equal(O.std_gate(I, Z, 5, 100.0), O.std_gate(I + 300, Z, 5, 100.0))


# -------------------------------------------------------- hybrid median ----
def test_hm_constant_and_impulse():
    """constant unchanged; a single impulse is removed."""
    E = np.full((9, 9), 77, np.uint16)
    np.testing.assert_array_equal(O.hybrid_median(E), E)
    E = np.zeros((9, 9), np.uint16)
    E[4, 4] = 255
    assert not O.hybrid_median(E).any()


def test_hm_keeps_thin_line_plain_median_erases_it():
    """SPEC.md:223 / PAPER.md:40: a 1-px line survives the hybrid median but not
    a plain 5x5 median (5 of 25 on-line)."""
    E = np.zeros((15, 15), np.uint16)
    E[7, :] = 100
    hm = O.hybrid_median(E)
    assert (hm[7, :] == 100).all() and hm.sum() == 100 * 15
    plain = ndi.median_filter(E, size=5, mode="nearest")
    assert not plain.any()
    D = np.zeros((15, 15), np.uint16)
    np.fill_diagonal(D, 100)
    assert (np.diag(O.hybrid_median(D))[2:-2] == 100).all()


def _hm_brute(E, m):
    H, W = E.shape
    R = m // 2
    out = np.zeros_like(E)
    at = lambda y, x: int(E[min(max(y, 0), H - 1), min(max(x, 0), W - 1)])
    for y in range(H):
        for x in range(W):
            plus = [at(y, x)] + [at(y, x + d) for d in range(-R, R + 1) if d] + \
                   [at(y + d, x) for d in range(-R, R + 1) if d]
            cross = [at(y, x)] + [at(y + d, x + d) for d in range(-R, R + 1) if d] + \
                    [at(y + d, x - d) for d in range(-R, R + 1) if d]
            out[y, x] = statistics.median([statistics.median(plus), statistics.median(cross),
                                           at(y, x)])
    return out


@pytest.mark.parametrize("m", [3, 5, 7])
def test_hm_brute_force(m):
    rng = np.random.default_rng(7 + m)
    for _ in range(4):
        E = rng.integers(0, 6, (9, 11)).astype(np.uint16) * 50
        E[rng.random(E.shape) < 0.4] = 0
        np.testing.assert_array_equal(O.hybrid_median(E, m), _hm_brute(E, m))


@pytest.mark.parametrize("m1,m2", [(5, 3), (3, 5), (7, 7), (5, 5)])
def test_two_level_hm_is_the_composition(m1, m2):
    """the water pipeline passes the merged image "through a hybrid
    median filter in multiple levels"; reading R17 makes level 2 the same filter
    (window m2, replicate padding) applied to level 1's output.  Checked against
    the independent brute force applied twice to the oracle's merged image E."""
    rng = np.random.default_rng(40 + m1 * 8 + m2)
    I = scenes.random_image(rng, 13, 17, 8)
    p = O.Params(bit_depth=8, median_window=m1, median_window2=m2, zc_threshold=(0.005, 0.0))
    res = O.run(I, p, intermediates=True)
    np.testing.assert_array_equal(res.out, _hm_brute(_hm_brute(res.E, m1), m2))
    # the single-level run shares E and differs only in the last filter
    one = O.run(I, O.Params(bit_depth=8, median_window=m1, zc_threshold=(0.005, 0.0)))
    np.testing.assert_array_equal(one, _hm_brute(res.E, m1))


def test_two_level_hm_keeps_thin_lines():
    """The hybrid median's line preservation holds at every
    level: a 1-px horizontal and a 1-px diagonal line survive 5 then 3."""
    E = np.zeros((17, 17), np.uint16)
    E[8, :] = 90
    np.fill_diagonal(E, 90)
    two = _hm_brute(_hm_brute(E, 5), 3)
    assert (two[8, :] == 90).all()
    assert (np.diag(two)[2:-2] == 90).all()


def test_hm_output_values_come_from_window():
    rng = np.random.default_rng(8)
    E = rng.integers(0, 1000, (12, 12)).astype(np.uint16)
    out = O.hybrid_median(E)
    P = np.pad(E, 2, mode="edge")
    for y in range(12):
        for x in range(12):
            assert out[y, x] in P[y:y + 5, x:x + 5]


# ------------------------------------------------------------- pipeline ----
def test_pipeline_constant_image_is_empty():
    for b in (8, 10):
        I = np.full((20, 30), 37, np.uint8 if b == 8 else np.uint16)
        assert not O.run(I, O.Params(bit_depth=b)).any()


def test_pipeline_block_fixture_is_localised():
    """a bright 8x8 block -> non-empty output within 4 px of its edge."""
    I = np.full((64, 64), 20, np.uint8)
    I[28:36, 28:36] = 200
    for hm in (False, True):
        out = O.run(I, O.Params(bit_depth=8, hybrid_median=hm, out_mode=1))
        ys, xs = np.nonzero(out)
        assert ys.size > 0
        assert ys.min() >= 24 and ys.max() <= 39 and xs.min() >= 24 and xs.max() <= 39
        inner = out[32 - 0:32 + 0 + 1, 32:33]
        assert not inner.any()


def test_pipeline_merge_contains_each_branch_and_is_branch_symmetric():
    I = scenes.scene_c1(size=96)
    p = O.Params(bit_depth=8, hybrid_median=False, out_mode=1)
    res = O.run(I, p, intermediates=True)
    M = res.out > 0
    assert (M >= (res.keep[0] > 0)).all() and (M >= (res.keep[1] > 0)).all()
    ps = O.Params(bit_depth=8, hybrid_median=False, out_mode=1, sigma=(20.0, 0.5))
    np.testing.assert_array_equal(O.run(I, ps), res.out)


def _pipeline_cases():
    yield O.Params(bit_depth=8)
    yield O.Params(bit_depth=8, out_mode=1, zc_threshold=(0.02, 0.01))
    yield O.Params(bit_depth=10, std_source=1, std_threshold=(20.0, 40.0), std3_threshold=(10.0, -1.0))
    yield O.Params(bit_depth=12, log_size=(3, 7), std_window=3, median_window=3)
    yield O.Params(bit_depth=8, median_window=5, median_window2=3, zc_threshold=(0.01, 0.0))


@pytest.mark.parametrize("pi", range(5))
def test_pipeline_dihedral_covariance(pi):
    """Masks are 8-fold symmetric, N4 / square windows / +,x groups are dihedral
    invariant and replicate padding commutes: f(T I) = T f(I)."""
    p = list(_pipeline_cases())[pi]
    rng = np.random.default_rng(10 + pi)
    I = scenes.random_image(rng, 29, 37, p.bit_depth)
    out = O.run(I, p)
    for T in _DIHEDRAL:
        np.testing.assert_array_equal(O.run(np.ascontiguousarray(T(I)), p), T(out))


def test_pipeline_negation_keeps_the_kept_set():
    """I -> M - I negates every LoG response exactly (zero-sum masks); R* and
    both std sources are sign-symmetric, so the 0/255 output is unchanged."""
    rng = np.random.default_rng(11)
    for b, src in [(8, 0), (10, 0), (10, 1)]:
        p = O.Params(bit_depth=b, out_mode=1, std_source=src,
                     std_threshold=(0.3, 0.3) if src == 0 else (30.0, 30.0))
        I = scenes.random_image(rng, 40, 33, b)
        M = (1 << b) - 1
        Ineg = (M - I.astype(np.int64)).astype(I.dtype)
        np.testing.assert_array_equal(O.run(Ineg, p), O.run(I, p))


@pytest.mark.parametrize("hm,m2,halo", [(True, 0, 7), (False, 0, 5), (True, 3, 8), (True, 7, 10)])
def test_pipeline_strip_invariance_with_halo(hm, m2, halo):
    """Row strips with `halo` real rows above/below (clamping only at the true
    image edge) reproduce the whole-image result: the dependency cone of an
    output row is LoG 2 + ZC 1 + std 2 (+ HM 2) (+ second HM level m2 // 2)
    rows."""
    I = scenes.scene_c1(size=128)
    p = O.Params(bit_depth=8, hybrid_median=hm, median_window2=m2, zc_threshold=(0.01, 0.01))
    whole = O.run(I, p)
    H = I.shape[0]
    for a, b in [(0, 9), (9, 40), (40, 41), (41, 100), (100, 128), (57, 64)]:
        lo, hi = max(0, a - halo), min(H, b + halo)
        part = O.run(np.ascontiguousarray(I[lo:hi]), p)
        np.testing.assert_array_equal(part[a - lo:a - lo + (b - a)], whole[a:b])


def test_pipeline_rejects_out_of_range_pixels():
    I = np.full((4, 4), 300, np.uint16)
    with pytest.raises(ValueError):
        O.run(I, O.Params(bit_depth=8))


# ------------------------------------------- adaptive thresholds (NEXT-2) ----
def test_global_std_is_the_exact_formula():
    """R21: sigma = sqrt(n*S2 - S1^2) / n with the integer numerator exact and
    rounded once.  Python ints are exact and float(int) / math.sqrt round
    correctly, so the oracle must agree bit for bit -- including numerators
    far beyond 2^64 (the 128-bit path)."""
    rng = np.random.default_rng(21)
    cases = [(1, 5, 25), (4, 2, 2), (3, 6, 14), (2, 0, 2 * (2**24 - 1) ** 2)]
    for _ in range(300):
        n = int(rng.integers(1, 2**31))
        v = int(rng.integers(0, 2**24))
        s1 = int(rng.integers(-n, n)) * v // 7
        s2 = n * v * v  # >= s1^2 / n
        cases.append((n, s1, s2))
    for n, s1, s2 in cases:
        want = math.sqrt(float(n * s2 - s1 * s1)) / float(n)
        assert O.global_std(n, s1, s2) == want, (n, s1, s2)


def test_std_of_response_and_intensity_match_numpy():
    rng = np.random.default_rng(22)
    r = rng.integers(-(2**24) + 1, 2**24, (37, 53)).astype(np.int64)
    assert math.isclose(O.std_of_response(r), float(np.std(r.astype(np.float64))), rel_tol=1e-12)
    I = rng.integers(0, 65536, (29, 31)).astype(np.uint16)
    assert math.isclose(O.std_of_intensity(I), float(np.std(I.astype(np.float64))), rel_tol=1e-12)
    # closed form: half a, half b -> sigma = |a - b| / 2 exactly; constant -> 0
    two = np.array([[100, 900] * 8] * 3, np.uint16)
    assert O.std_of_intensity(two) == 400.0
    assert O.std_of_intensity(np.full((5, 5), 77, np.uint16)) == 0.0
    assert O.std_of_response(np.zeros((4, 4), np.int64)) == 0.0


def _thr_for(t, F, b):
    """A normalised absolute ZC threshold whose integer threshold is exactly t."""
    return (t - 0.5) / (2.0**F * ((1 << b) - 1)) if t > 0 else 0.0


@pytest.mark.parametrize("b,k", [(8, 0.75), (10, 0.3), (12, 1.0), (8, 0.05)])
def test_adaptive_zc_threshold_equals_absolute_with_that_t(b, k):
    """t_j = ceil(k * global std of r_j).  The expected t comes from
    scipy's correlate and numpy's std; the adaptive pipeline must then equal the
    absolute-threshold pipeline at that integer t."""
    rng = np.random.default_rng(23 + b)
    I = scenes.random_image(rng, 41, 47, b)
    ts, thr = [], []
    for j, s in enumerate((0.5, 20.0)):
        q, F = O.mask_int(s, 5, b)
        r = ndi.correlate(I.astype(np.int64), q.astype(np.int64), mode="nearest")
        x = k * float(np.std(r.astype(np.float64)))
        assert abs(x - round(x)) > 1e-6  # not on a rounding boundary
        ts.append(math.ceil(x))
        thr.append(_thr_for(ts[-1], F, b))
        assert O.adaptive_zc_threshold(k, O.std_of_response(r)) == ts[-1]
    pa = O.Params(bit_depth=b, zc_threshold=(k, k), adaptive=1, out_mode=1)
    pb = O.Params(bit_depth=b, zc_threshold=tuple(thr), out_mode=1)
    np.testing.assert_array_equal(O.run(I, pa), O.run(I, pb))


def test_adaptive_std_threshold_equals_absolute_with_that_T():
    """std thresholds = k * global intensity std (INTENSITY source)."""
    rng = np.random.default_rng(24)
    I = scenes.random_image(rng, 45, 39, 10)
    v = I.astype(np.int64).ravel()
    sI = O.global_std(v.size, int(v.sum()), int((v * v).sum()))
    k, k3 = (0.8, 1.3), (1.5, -1.0)
    pa = O.Params(bit_depth=10, std_source=1, std_threshold=k, std3_threshold=k3, adaptive=2, out_mode=1)
    pb = O.Params(bit_depth=10, std_source=1, std_threshold=(k[0] * sI, k[1] * sI),
                  std3_threshold=(k3[0] * sI, -1.0), out_mode=1)
    np.testing.assert_array_equal(O.run(I, pa), O.run(I, pb))


def test_adaptive_constant_image_and_invariances():
    """Constant image: sigma = 0 -> t = 0, still empty.  The global stds are
    invariant under the dihedral maps and I -> M - I, so the covariance pins of
    the absolute pipeline carry over."""
    assert not O.run(np.full((20, 20), 9, np.uint8), O.Params(bit_depth=8, adaptive=1, zc_threshold=(0.7, 0.7))).any()
    rng = np.random.default_rng(25)
    I = scenes.random_image(rng, 33, 28, 8)
    p = O.Params(bit_depth=8, adaptive=1, zc_threshold=(0.6, 0.9), out_mode=1)
    out = O.run(I, p)
    for T in _DIHEDRAL:
        np.testing.assert_array_equal(O.run(np.ascontiguousarray(T(I)), p), T(out))
    np.testing.assert_array_equal(O.run((255 - I.astype(np.int64)).astype(np.uint8), p), out)


# ------------------------------------------------ F32 mode + response std (NEXT-3) ----
@pytest.mark.parametrize("sigma,n,b", [(0.5, 5, 8), (20.0, 5, 10), (1.4, 7, 12), (0.8, 3, 16)])
def test_log_f32_matches_scipy_and_snaps(sigma, n, b):
    """R23: r^ = (sum w I) / (M c) with w = (float) L_dc; |r^| < 1e-4 -> 0.
    scipy's correlate (double) of the same float weights is the reference."""
    w, c = O.mask_f32(sigma, n)
    L = O.log_dc(sigma, n)
    assert np.array_equal(w, L.astype(np.float32)) and c == abs(L[n // 2, n // 2])
    rng = np.random.default_rng(int(sigma * 10) + n + b)
    I = scenes.random_image(rng, 23, 29, b)
    M = (1 << b) - 1
    rh = O.log_response_f(I, w, 1.0 / (M * c))
    ref = ndi.correlate(I.astype(np.float64), w.astype(np.float64), mode="nearest") * (1.0 / (M * c))
    ref[np.abs(ref) < 1e-4] = 0.0
    np.testing.assert_allclose(rh, ref, rtol=1e-12, atol=1e-15)
    # a constant image: the float mask sums to ~0, so every response snaps to exactly 0
    assert not O.log_response_f(np.full((9, 9), M, I.dtype), w, 1.0 / (M * c)).any()


def test_zc_f32_equals_integer_rule_on_integer_values():
    """The float rule R* evaluated on integer-valued responses is the integer
    rule (exhaustive 5-pixel crosses, as the integer pin)."""
    vals = [-3, -1, 0, 1, 3]
    for t in (0, 2, 4, 5):
        pats = np.array(list(itertools.product(vals, repeat=5)), np.float64)
        for i, (c, u, d, l, rr) in enumerate(pats):
            R = np.zeros((3, 3))
            R[1, 1], R[0, 1], R[2, 1], R[1, 0], R[1, 2] = c, u, d, l, rr
            R[0, 0], R[0, 2], R[2, 0], R[2, 2] = u, u, d, d
            Zf = O.zero_crossing_f(R, float(t))
            assert Zf[1, 1] == _zc_brute(int(c), [int(u), int(d), int(l), int(rr)], t)


def _stdev_gate_brute(r, Z, w, T, T3, at_zc):
    """Eq. 2 literally with exact rationals: keep = Z & s_w > T & (T3<0 | s_3 > T3)."""
    from fractions import Fraction as Fr
    H, W = Z.shape
    keep = np.zeros_like(Z)
    at = lambda y, x: (0 if at_zc and not Z[min(max(y, 0), H - 1), min(max(x, 0), W - 1)]
                       else int(r[min(max(y, 0), H - 1), min(max(x, 0), W - 1)]))

    def var_gt(vals, T):  # sample variance > T^2, exactly
        n = len(vals)
        m = Fr(sum(vals), n)
        return sum((Fr(v) - m) ** 2 for v in vals) / (n - 1) > Fr(T) ** 2
    for y in range(H):
        for x in range(W):
            if not Z[y, x]:
                continue
            R = w // 2
            ok = var_gt([at(y + dy, x + dx) for dy in range(-R, R + 1) for dx in range(-R, R + 1)], T)
            if ok and T3 >= 0:
                ok = var_gt([at(y + dy, x + dx) for dy in (-1, 0, 1) for dx in (-1, 0, 1)], T3)
            keep[y, x] = ok
    return keep


@pytest.mark.parametrize("w,at_zc", [(5, False), (5, True), (3, False), (7, True)])
def test_std_gate_response_brute_force(w, at_zc):
    """R24: Eq. 2 over the signed response window (or the response
    at crossings), integer path exact against rational arithmetic."""
    rng = np.random.default_rng(50 + w + at_zc)
    r = rng.integers(-900, 900, (11, 13)).astype(np.int64)
    Z = (rng.random((11, 13)) < 0.5).astype(np.uint8)
    for T, T3 in [(300.3, -1.0), (450.7, 200.1), (0.0, -1.0), (700.2, 650.9)]:
        got = O.std_gate_response(r, Z, w, T, T3, at_zc)
        np.testing.assert_array_equal(got, _stdev_gate_brute(r, Z, w, T, T3, at_zc), err_msg=f"T={T} T3={T3}")
        gf = O.std_gate_response(r.astype(np.float64), Z, w, T, T3, at_zc)  # the float variant agrees here
        np.testing.assert_array_equal(gf, got)


def test_pipeline_f32_agrees_with_integer_mode_away_from_ties():
    """INT and F32 modes quantise the same Eq. 1 masks differently; their outputs
    must agree almost everywhere (a sign error, scale error or dropped term in
    either path would break this massively)."""
    img = scenes.scene_c1(clean=False)
    for src, T in [(0, (0.3, 0.3)), (2, (0.02, 0.02))]:
        pi = O.Params(bit_depth=8, zc_threshold=(0.01, 0.01), out_mode=1, std_source=src, std_threshold=T)
        pf = O.Params(bit_depth=8, zc_threshold=(0.01, 0.01), out_mode=1, std_source=src, std_threshold=T,
                      mask_mode=1)
        a, b = O.run(img, pi), O.run(img, pf)
        assert a.any() and (a != b).mean() < 0.01, (src, (a != b).mean())
    # the float responses are the integer ones rescaled (within the quantisation error)
    res_i = O.run(img, pi, intermediates=True)
    res_f = O.run(img, pf, intermediates=True)
    for j, s in enumerate((0.5, 20.0)):
        _, F = O.mask_int(s, 5, 8)
        scaled = res_i.r[j] / (2.0**F * 255)
        assert np.max(np.abs(scaled - res_f.r[j])) < 2e-3 * np.max(np.abs(scaled))


def test_pipeline_response_std_source_matches_stagewise_composition():
    """std_source 2/3 in the pipeline = LoG -> ZC -> std_gate_response with the
    threshold converted to integer units T * 2^F * M (R9 normalisation)."""
    rng = np.random.default_rng(60)
    I = scenes.random_image(rng, 31, 37, 10)
    for src in (2, 3):
        p = O.Params(bit_depth=10, std_source=src, std_threshold=(0.05, 0.01), hybrid_median=False,
                     zc_threshold=(0.002, 0.0), out_mode=1)
        res = O.run(I, p, intermediates=True)
        for j, s in enumerate((0.5, 20.0)):
            _, F = O.mask_int(s, 5, 10)
            unit = 2.0**F * 1023
            k = O.std_gate_response(res.r[j], res.z[j], 5, p.std_threshold[j] * unit, -1.0, src == 3)
            np.testing.assert_array_equal(k, res.keep[j])


# ------------------------------------- pins added in round 2 ----
@pytest.mark.parametrize("w", [3, 5, 7])
def test_std_gate_windows_3_5_7_vs_statistics_stdev(w):
    """lfo_std_gate at every window side against Eq. 2 evaluated by
    statistics.stdev on the replicate-padded w x w window of each crossing pixel
    (intensity source and binary source; with and without the 3x3 re-check of
    PAPER.md:94).  Thresholds are drawn away from the deviations' values so the
    strict '>' is decided the same way by the exact and the float route."""
    import statistics
    rng = np.random.default_rng(700 + w)
    for binary in (False, True):
        H, W = 19, 23
        src = (rng.integers(0, 2, (H, W)) if binary else rng.integers(0, 1024, (H, W))).astype(np.uint16)
        Z = (rng.random((H, W)) < 0.5).astype(np.uint8)
        P = np.pad(src.astype(float), w // 2, mode="edge")
        P3 = np.pad(src.astype(float), 1, mode="edge")
        s_all = [statistics.stdev(P[y:y + w, x:x + w].ravel().tolist()) for y in range(H) for x in range(W)]
        s3_all = [statistics.stdev(P3[y:y + 3, x:x + 3].ravel().tolist()) for y in range(H) for x in range(W)]
        vals = sorted(set(round(v, 9) for v in s_all))
        T = (vals[len(vals) // 3] + vals[len(vals) // 3 + 1]) / 2  # between two attained values
        v3 = sorted(set(round(v, 9) for v in s3_all))
        T3 = (v3[len(v3) // 4] + v3[len(v3) // 4 + 1]) / 2
        for t3 in (-1.0, T3):
            keep = O.std_gate(src, Z, w, T, t3)
            for y in range(H):
                for x in range(W):
                    k = y * W + x
                    want = bool(Z[y, x]) and s_all[k] > T and (t3 < 0 or s3_all[k] > t3)
                    assert bool(keep[y, x]) == want, (w, binary, t3, y, x, s_all[k], T)


def test_zc_threshold_int_exact_product():
    """R9: t = ceil(thr * 2^F * (2^b - 1)), pinned to an exact rational
    evaluation (fractions.Fraction of the double thr: no rounding anywhere),
    for thresholds whose exact product is not within 1e-6 of an integer (there
    the double evaluation is the definition and both must agree)."""
    from fractions import Fraction
    rng = np.random.default_rng(77)
    checked = 0
    for b in (1, 8, 10, 12, 16):
        for s in (0.5, 20.0):
            _, F = O.mask_int(s, 5, b)
            for thr in list(rng.random(200) * 0.2) + [0.0, 0.01, 0.02, 0.05, 0.3]:
                exact = Fraction(float(thr)) * (2 ** F) * (2 ** b - 1)
                if thr > 0 and abs(exact - round(exact)) < Fraction(1, 10**6):
                    continue
                want = math.ceil(exact)
                assert O.zc_threshold_int(float(thr), F, b) == want, (b, s, thr)
                checked += 1
    assert checked > 1500
