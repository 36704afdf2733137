"""CPU-only checks of the C-ABI library: it loads, exports every declared
symbol, validates parameters synchronously, and its host-side mask synthesis
equals the oracle's independent one.  No compute call needs a GPU here."""
import ctypes
import math
import os
import re
import subprocess

import numpy as np
import pytest

import oracle as O
from paper_1304_3992_b200 import build as B
from paper_1304_3992_b200 import lfe

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def _built():
    B.build()
    lfe.load()


def _declared(header):
    text = open(os.path.join(ROOT, "include", header)).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(lfe_[a-z0-9_]+)\s*\(", text)))


def _exported(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", lib], capture_output=True, text=True).stdout
    return set(re.findall(r"\bT (lfe_\w+)", out))


def test_exports_every_declared_symbol():
    """liblfe.so exports exactly lfe.h's calls; the test-only entries of
    lfe_test.h live in the separate liblfe_test.so."""
    prod, test = _exported(B.LIB), _exported(B.TEST_LIB)
    declared, declared_test = _declared("lfe.h"), _declared("lfe_test.h")
    assert declared and declared_test, "no declarations parsed"
    assert sorted(prod) == declared, sorted(set(prod) ^ set(declared))
    assert sorted(test) == declared_test, sorted(set(test) ^ set(declared_test))
    assert sorted(lfe.EXPORTS) == declared
    assert sorted(lfe.TEST_EXPORTS) == declared_test


def test_test_library_loads_against_the_product():
    T = lfe.load_test()
    for name in lfe.TEST_EXPORTS:
        assert hasattr(T, name)


def test_no_torch_types_in_signatures():
    for h in ("lfe.h", "lfe_test.h"):
        text = open(os.path.join(ROOT, "include", h)).read()
        assert "torch" not in text.replace("torch.distributed", "") or "Tensor" not in text
        assert "at::" not in text and "c10" not in text


def test_abi_version_and_params_default():
    assert lfe.lfe_abi_version() == 1
    p = lfe.lfe_params_default()
    assert p.abi_size == ctypes.sizeof(lfe.lfe_params) == 120
    assert (p.bit_depth, p.sigma[0], p.sigma[1], p.log_size[0], p.log_size[1]) == (8, 0.5, 20.0, 5, 5)
    assert (p.std_source, p.std_window, p.std_threshold[0], p.std3_threshold[0]) == (0, 5, 0.3, -1.0)
    assert (p.hybrid_median, p.median_window, p.out_mode, p.median_window2) == (1, 5, 0, 0)
    assert lfe.lfe_test_validate(p) == lfe.LFE_OK
    # the Python mirror of the defaults is the same struct
    q = lfe.Params().to_c()
    assert bytes(q) == bytes(p)


def _with(**kw):
    p = lfe.lfe_params_default()
    for k, v in kw.items():
        if isinstance(v, tuple):
            arr = getattr(p, k)
            arr[0], arr[1] = v
        else:
            setattr(p, k, v)
    return p


@pytest.mark.parametrize("kw,status", [
    (dict(abi_size=100), lfe.LFE_EINVAL),
    (dict(bit_depth=0), lfe.LFE_EINVAL),
    (dict(bit_depth=17), lfe.LFE_EINVAL),
    (dict(sigma=(0.0, 20.0)), lfe.LFE_EINVAL),
    (dict(sigma=(0.5, -1.0)), lfe.LFE_EINVAL),
    (dict(sigma=(float("nan"), 1.0)), lfe.LFE_EINVAL),
    (dict(sigma=(float("inf"), 1.0)), lfe.LFE_EINVAL),
    (dict(log_size=(4, 5)), lfe.LFE_EINVAL),
    (dict(log_size=(5, 11)), lfe.LFE_EUNSUPPORTED),
    (dict(log_size=(1, 5)), lfe.LFE_EUNSUPPORTED),
    (dict(zc_threshold=(-0.1, 0.0)), lfe.LFE_EINVAL),
    (dict(std_window=4), lfe.LFE_EINVAL),
    (dict(std_window=9), lfe.LFE_EUNSUPPORTED),
    (dict(std_threshold=(-1.0, 0.3)), lfe.LFE_EINVAL),
    (dict(std3_threshold=(float("nan"), -1.0)), lfe.LFE_EINVAL),
    (dict(hybrid_median=2), lfe.LFE_EINVAL),
    (dict(median_window=6), lfe.LFE_EINVAL),
    (dict(median_window=11), lfe.LFE_EUNSUPPORTED),
    (dict(out_mode=3), lfe.LFE_EINVAL),
    (dict(adaptive=4), lfe.LFE_EINVAL),
    (dict(mask_mode=2), lfe.LFE_EINVAL),
    (dict(reserved1=1), lfe.LFE_EINVAL),
    (dict(std_source=4), lfe.LFE_EINVAL),
    (dict(mask_mode=1, adaptive=1), lfe.LFE_EINVAL),  # adaptive ZC is defined on integer responses
    (dict(adaptive=2), lfe.LFE_EINVAL),  # LFE_ADAPT_STD needs the intensity source
    (dict(median_window2=4), lfe.LFE_EINVAL),
    (dict(median_window2=-3), lfe.LFE_EINVAL),
    (dict(median_window2=9), lfe.LFE_EUNSUPPORTED),
    (dict(median_window2=1), lfe.LFE_EUNSUPPORTED),
    (dict(hybrid_median=0, median_window2=3), lfe.LFE_EINVAL),
])
def test_validation_errors(kw, status):
    p = _with(**kw)
    assert lfe.lfe_test_validate(p) == status
    with pytest.raises(lfe.LfeError) as ei:
        lfe.lfe_create(p)
    assert ei.value.status == status  # validation precedes the device check


def test_create_without_gpu_is_enodev():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    with pytest.raises(lfe.LfeError) as ei:
        lfe.lfe_create(lfe.lfe_params_default())
    assert ei.value.status == lfe.LFE_ENODEV


def test_strerror():
    for s in range(7):
        assert lfe.lfe_strerror(s)
    assert lfe.lfe_strerror(99) == "unknown status"


@pytest.mark.parametrize("sigma", [0.5, 0.7, math.sqrt(0.5), 1.0, 1.7, 4.0, math.sqrt(20), 20.0, 55.0])
@pytest.mark.parametrize("n", [3, 5, 7, 9])
@pytest.mark.parametrize("b", [1, 4, 8, 10, 12, 14, 16])
def test_library_masks_equal_oracle_masks(sigma, n, b):
    """Two independent implementations of reading R3 agree exactly."""
    q_lib, F_lib = lfe.lfe_test_mask(sigma, n, b)
    q_or, F_or = O.mask_int(sigma, n, b)
    assert F_lib == F_or
    np.testing.assert_array_equal(q_lib, q_or)
