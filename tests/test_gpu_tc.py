"""GPU parity of the fused kernel's tensor-core LoG (tcgen05) against
the CPU oracle and against the same kernel with the LoG forced onto the CUDA cores
(LFE_OPT_LOG_UNIT), bit for bit.

The tensor-core path is exact when the u16 input bits read as fp16 equal v * 2^-24
(v < 2048, b <= 11; b = 12 splits v into v & 0x7FF and bit 11) and every mask
coefficient is an fp16 value; the cases below
cover every compiled TC variant family (median levels 0/1/2, extract / mask, with /
without the gap test, the 3x3 re-check), the walks it takes (interior, cheap column
edges, and the CUDA-core fallbacks inside the same kernel: edge rows and widths
that are not a multiple of 4), the largest 11- and 12-bit values (the first fp16
binade, bit 11, and the largest partial sums R3 allows) and the piece / chunk boundaries of the MMA
pipeline (rows per piece, 8-row chunks, 4-row MMA halves).
"""
import itertools

import numpy as np
import pytest

import oracle as O
from paper_1304_3992_b200 import lfe, scenes
from test_gpu_parity import _oparams, _pitched, assert_same

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    lfe.load()


def run(img, p, log_unit=lfe.LFE_LOG_TENSOR_CORES, seg=0):
    with lfe.Context(p) as ctx:
        ctx.set_option(lfe.LFE_OPT_KERNEL, lfe.LFE_KERNEL_FUSED)
        ctx.set_option(lfe.LFE_OPT_LOG_UNIT, log_unit)
        if seg:
            ctx.set_option(lfe.LFE_OPT_TILE_H, seg)
        tin = torch.uint8 if p.bit_depth <= 8 else torch.uint16
        tout = torch.uint8 if p.out_mode == lfe.LFE_OUT_MASK else tin
        d = _pitched(img.shape, tin)
        d.copy_(torch.from_numpy(np.ascontiguousarray(img)))
        out = _pitched(img.shape, tout)
        ctx.extract(d, out)
        ctx.check()
        return out.cpu().numpy()


def _variants():
    yield lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02))                        # c3's variant
    yield lfe.Params(bit_depth=10, zc_threshold=(0.0, 0.0))                          # no gap test
    yield lfe.Params(bit_depth=11, zc_threshold=(0.01, 0.0), out_mode=lfe.LFE_OUT_MASK)
    yield lfe.Params(bit_depth=9, hybrid_median=False, zc_threshold=(0.02, 0.01))
    yield lfe.Params(bit_depth=10, hybrid_median=False, out_mode=lfe.LFE_OUT_MASK)
    yield lfe.Params(bit_depth=10, median_window2=3, zc_threshold=(0.01, 0.01))      # two median levels
    yield lfe.Params(bit_depth=11, median_window2=3, out_mode=lfe.LFE_OUT_MASK)
    yield lfe.Params(bit_depth=10, std3_threshold=(0.4, 0.2), zc_threshold=(0.01, 0.0))  # 3x3 re-check
    yield lfe.Params(bit_depth=10, std3_threshold=(0.3, 0.3), hybrid_median=False, out_mode=lfe.LFE_OUT_MASK)
    yield lfe.Params(bit_depth=10, sigma=(1.0, 2.0), zc_threshold=(0.005, 0.02))   # other masks
    # b = 12 (c4): the patch split into its low 11 bits and bit 11 (TC12)
    yield lfe.Params(bit_depth=12, zc_threshold=(0.02, 0.02))
    yield lfe.Params(bit_depth=12, zc_threshold=(0.0, 0.0), out_mode=lfe.LFE_OUT_MASK)
    yield lfe.Params(bit_depth=12, median_window2=3, zc_threshold=(0.01, 0.01))
    yield lfe.Params(bit_depth=12, std3_threshold=(0.4, 0.2), zc_threshold=(0.01, 0.0))
    yield lfe.Params(bit_depth=12, hybrid_median=False, zc_threshold=(0.02, 0.0))
    # u8 (c1, c2): bytes as u16 pairs, weights as fp16(q) + remainder (TC8)
    yield lfe.Params(bit_depth=8, zc_threshold=(0.02, 0.02))
    yield lfe.Params(bit_depth=8, zc_threshold=(0.0, 0.0), out_mode=lfe.LFE_OUT_MASK)
    yield lfe.Params(bit_depth=8, median_window2=3, zc_threshold=(0.01, 0.01))
    yield lfe.Params(bit_depth=8, std3_threshold=(0.4, 0.2), zc_threshold=(0.01, 0.0))
    yield lfe.Params(bit_depth=8, hybrid_median=False, zc_threshold=(0.02, 0.0))
    yield lfe.Params(bit_depth=6, sigma=(1.0, 2.0), zc_threshold=(0.01, 0.02))


VARIANTS = list(_variants())
# W % 4 == 0 widths take the cheap column-edge walk on the tensor cores, other widths
# the general fix-up walk on the CUDA cores; 1344 = one CTA column group, 2700 three
SHAPES = [(40, 64), (64, 124), (33, 1344), (70, 1348), (29, 2700), (120, 517), (9, 300), (200, 96)]


@pytest.mark.parametrize("vi", range(len(VARIANTS)))
def test_tc_equals_cuda_cores_and_oracle(vi):
    p = VARIANTS[vi]
    rng = np.random.default_rng(4200 + vi)
    for (H, W), kind in itertools.product(SHAPES, ["mixed", "blocks"]):
        img = scenes.random_image(rng, H, W, p.bit_depth, kind)
        want = O.run(img, _oparams(p))
        got = run(img, p)
        assert_same(got, want, f"TC {H}x{W} {kind} {p}")
        assert_same(run(img, p, lfe.LFE_LOG_CUDA_CORES), got, f"CUDA cores vs TC {H}x{W} {kind}")


@pytest.mark.parametrize("bd", [8, 11, 12])
@pytest.mark.parametrize("kind", ["max", "binade", "checker", "ramp"])
def test_tc_bit_depth_extremes(kind, bd):
    """b = 11: the u16 bits 1024..2047 are fp16 normals of the first binade (still
    v * 2^-24); b = 12: values 2048..4095 take the bit-11 part (TC12); the largest
    partial sums R3 admits (M * sum|q| < 2^24) come from checkerboards of 0 and the
    maximum under the mask's sign pattern."""
    H, W = 96, 1348
    rng = np.random.default_rng(11)
    y, x = np.mgrid[0:H, 0:W]
    M = (1 << bd) - 1
    if kind == "max":
        img = np.where(rng.random((H, W)) < 0.5, M, 0)
    elif kind == "binade":
        img = rng.integers((M + 1) // 2, M + 1, (H, W))
    elif kind == "checker":
        img = np.where(((y // 2) + (x // 2)) % 2 == 0, M, 0)
    else:
        img = (x * 7 + y * 13) % (M + 1)
    img = img.astype(np.uint8 if bd <= 8 else np.uint16)
    for p in (lfe.Params(bit_depth=bd, zc_threshold=(0.0, 0.0)),
              lfe.Params(bit_depth=bd, zc_threshold=(0.02, 0.02), median_window2=3)):
        want = O.run(img, _oparams(p))
        assert_same(run(img, p), want, f"{kind} {p}")


@pytest.mark.parametrize("seg", [1, 3, 4, 5, 8, 9, 15, 16, 17, 100])
def test_tc_piece_and_chunk_boundaries(seg):
    """Pieces of every length around the 8-row chunk and the 4-row MMA half: the
    prologue (first chunk), the mid-chunk issue and the last partial chunk."""
    img = scenes.random_image(np.random.default_rng(77), 150, 2696, 10, "mixed")
    p = lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02))
    assert_same(run(img, p, seg=seg), O.run(img, _oparams(p)), f"seg {seg}")


def test_tc12_c4_bands_equal_cuda_cores():
    """c4's recipe (b = 12 multispectral bands) at 2048^2, every band, both LoG units."""
    img = scenes.scene_c4(size=2048)
    p = lfe.Params(bit_depth=12, zc_threshold=(0.02, 0.02))
    for b in range(img.shape[0]):
        got = run(img[b], p)
        assert_same(got, run(img[b], p, lfe.LFE_LOG_CUDA_CORES), f"c4 band {b}")
        assert_same(got, O.run(img[b], _oparams(p)), f"c4 band {b} vs oracle")


def test_tc12_wide_strip_equals_oracle():
    """A 500-row strip of c4's width (8192 = 6.1 column groups) of random 12-bit data."""
    img = scenes.random_image(np.random.default_rng(12), 500, 8192, 12, "mixed")
    p = lfe.Params(bit_depth=12, zc_threshold=(0.02, 0.02))
    got = run(img, p)
    assert_same(got, run(img, p, lfe.LFE_LOG_CUDA_CORES), "b12 strip")
    assert_same(got, O.run(img, _oparams(p)), "b12 strip vs oracle")


def test_tc8_c2_tile_equals_cuda_cores():
    """c2's recipe (u8 urban tile) at 1500^2 (two column groups, one mostly idle), both LoG units."""
    img = scenes.scene_c2(size=1500)
    p = lfe.Params(bit_depth=8, zc_threshold=(0.02, 0.02))
    got = run(img, p)
    assert_same(got, run(img, p, lfe.LFE_LOG_CUDA_CORES), "c2 tile")
    assert_same(got, O.run(img, _oparams(p)), "c2 tile vs oracle")


def test_tc_c3_strip_equals_cuda_cores():
    """The bench scene's recipe: 600 rows of c3 at full width, both LoG units."""
    img = scenes.scene_c3(height=600)
    p = lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02))
    got = run(img, p)
    assert_same(got, run(img, p, lfe.LFE_LOG_CUDA_CORES), "c3 strip")
    assert_same(got, O.run(img, _oparams(p)), "c3 strip vs oracle")


def test_log_unit_option_validation():
    with lfe.Context(lfe.Params(bit_depth=10)) as ctx:
        ctx.set_option(lfe.LFE_OPT_LOG_UNIT, lfe.LFE_LOG_CUDA_CORES)
        ctx.set_option(lfe.LFE_OPT_LOG_UNIT, lfe.LFE_LOG_TENSOR_CORES)
        ctx.set_option(lfe.LFE_OPT_LOG_UNIT, lfe.LFE_LOG_AUTO)
        with pytest.raises(lfe.LfeError):
            ctx.set_option(lfe.LFE_OPT_LOG_UNIT, 3)


def test_auto_log_unit_equals_forced_units_on_c1():
    """c1 (below the 32-rows-per-SM rule: CUDA cores under AUTO) gives the same
    result on either unit."""
    img = scenes.scene_c1()
    p = lfe.Params(bit_depth=8, zc_threshold=(0.02, 0.02))
    got = run(img, p, lfe.LFE_LOG_AUTO)
    assert_same(got, run(img, p, lfe.LFE_LOG_TENSOR_CORES), "c1 auto vs tensor cores")
    assert_same(got, O.run(img, _oparams(p)), "c1 vs oracle")
