"""Property-based pins of the oracle (hypothesis, derandomised): invariants the
paper's definitions imply for ANY image and parameter set, so a plausible slip
in one stage (a transposed neighbour, a wrong padding, a sign) breaks them.
CPU only; small images so the whole file runs in seconds."""
import numpy as np
import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

import oracle as O

SETTINGS = settings(max_examples=60, deadline=None, derandomize=True,
                    suppress_health_check=[HealthCheck.too_slow])

_DIHEDRAL = [lambda a: a, lambda a: a[::-1], lambda a: a[:, ::-1], lambda a: a.T, lambda a: np.rot90(a),
             lambda a: np.rot90(a, 2), lambda a: np.rot90(a, 3), lambda a: a[::-1].T]


@st.composite
def cases(draw):
    b = draw(st.sampled_from([1, 3, 8, 10, 12, 16]))
    H = draw(st.integers(1, 14))
    W = draw(st.integers(1, 14))
    seed = draw(st.integers(0, 2**31 - 1))
    rng = np.random.default_rng(seed)
    M = (1 << b) - 1
    kind = draw(st.sampled_from(["uniform", "blocks", "sparse"]))
    if kind == "uniform":
        img = rng.integers(0, M + 1, (H, W))
    elif kind == "blocks":
        img = np.kron(rng.integers(0, M + 1, ((H + 2) // 3, (W + 2) // 3)), np.ones((3, 3), int))[:H, :W]
    else:
        img = np.where(rng.random((H, W)) < 0.2, M, 0)
    img = img.astype(np.uint8 if b <= 8 else np.uint16)
    p = O.Params(
        bit_depth=b,
        sigma=(draw(st.sampled_from([0.5, 0.8, 1.4])), draw(st.sampled_from([2.0, 20.0]))),
        log_size=(draw(st.sampled_from([3, 5, 7])), draw(st.sampled_from([3, 5]))),
        zc_threshold=(draw(st.sampled_from([0.0, 0.01, 0.05])), draw(st.sampled_from([0.0, 0.02]))),
        std_source=draw(st.sampled_from([0, 1, 2, 3])),
        std_window=draw(st.sampled_from([3, 5, 7])),
        hybrid_median=draw(st.booleans()),
        median_window=draw(st.sampled_from([3, 5])),
        out_mode=draw(st.sampled_from([0, 1])),
    )
    if p.std_source == 1:
        p.std_threshold = (draw(st.sampled_from([0.0, 5.0, 50.0])),) * 2
    elif p.std_source >= 2:
        p.std_threshold = (draw(st.sampled_from([0.0, 0.01, 0.1])),) * 2
    if p.hybrid_median and draw(st.booleans()):
        p.median_window2 = draw(st.sampled_from([3, 5]))
    return img, p


@SETTINGS
@given(cases())
def test_dihedral_covariance(c):
    """8-fold symmetric masks, N4 / square windows / + and x groups and
    replicate padding all commute with the dihedral group: f(T I) = T f(I)."""
    img, p = c
    out = O.run(img, p)
    for T in _DIHEDRAL:
        np.testing.assert_array_equal(O.run(np.ascontiguousarray(T(img)), p), T(out))


@SETTINGS
@given(cases())
def test_output_values_and_mask_mode(c):
    """EXTRACT outputs are input values or 0 at every level of the pipeline
    (hybrid medians select existing values); MASK outputs are 0 / 255."""
    img, p = c
    out = O.run(img, p)
    if p.out_mode == 1:
        assert set(np.unique(out)) <= {0, 255}
    elif not p.hybrid_median:
        assert np.all((out == 0) | (out == img))
    else:
        assert set(np.unique(out)) <= set(np.unique(img)) | {0}


@SETTINGS
@given(cases())
def test_negation_keeps_the_kept_set(c):
    """I -> M - I negates every integer response exactly (zero-sum masks), so
    rule R*, every std source and the OR keep the same pixels (MASK mode)."""
    img, p = c
    p.out_mode = 1
    M = (1 << p.bit_depth) - 1
    neg = (M - img.astype(np.int64)).astype(img.dtype)
    np.testing.assert_array_equal(O.run(neg, p), O.run(img, p))


@SETTINGS
@given(cases(), st.integers(0, 13))
def test_row_strips_with_halo(c, cut):
    """Two row strips, each with the library's halo of real rows (clamped only
    at the true edges), reproduce the whole image."""
    img, p = c
    H = img.shape[0]
    a = min(cut, H)
    halo = max(p.log_size) // 2 + 1 + p.std_window // 2 + (
        p.median_window // 2 + p.median_window2 // 2 if p.hybrid_median else 0)
    whole = O.run(img, p)
    for lo, hi in [(0, a), (a, H)]:
        if hi <= lo:
            continue
        s0, s1 = max(0, lo - halo), min(H, hi + halo)
        part = O.run(np.ascontiguousarray(img[s0:s1]), p)
        np.testing.assert_array_equal(part[lo - s0:hi - s0], whole[lo:hi])


@SETTINGS
@given(cases())
def test_constant_image_is_empty(c):
    img, p = c
    const = np.full_like(img, img.flat[0])
    assert not O.run(const, p).any()


@pytest.mark.parametrize("m", [3, 5])
def test_hybrid_median_idempotent_on_its_fixed_points(m):
    """A constant image and a 1-px line are fixed points of the hybrid median."""
    E = np.zeros((11, 11), np.uint16)
    E[5, :] = 7
    np.testing.assert_array_equal(O.hybrid_median(E, m), E)
    np.testing.assert_array_equal(O.hybrid_median(np.full((6, 6), 3, np.uint16), m), np.full((6, 6), 3))
