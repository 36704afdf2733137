"""Thin Python binding of liblfe (include/lfe.h) -- argument marshalling only.

Every step of the hot path runs inside liblfe's CUDA kernels; this module only
turns torch tensors / numpy arrays into pointers, pitches and streams.  There
is no CPU fallback: if liblfe.so is missing or no sm_100 device is present the
calls raise.

Function names mirror the C ABI (``lfe_create``, ``lfe_extract``, ...); the
``Context`` class is a convenience wrapper over them.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("LFE_LIB") or os.path.join(_PKG, "liblfe.so")  # LFE_LIB: A/B experiments only
# include/lfe_test.h: test-only entry points (LFE_TEST_LIB: an instrumented build, sanitizer runs only)
TEST_LIB_PATH = os.environ.get("LFE_TEST_LIB") or os.path.join(_PKG, "liblfe_test.so")

LFE_OK, LFE_EINVAL, LFE_EUNSUPPORTED, LFE_ENOMEM, LFE_ENODEV, LFE_ECUDA, LFE_ERANGE = range(7)
LFE_STD_ZC, LFE_STD_INTENSITY, LFE_STD_RESPONSE, LFE_STD_RESPONSE_AT_ZC = 0, 1, 2, 3
LFE_MASK_INT, LFE_MASK_F32 = 0, 1
LFE_OUT_EXTRACT, LFE_OUT_MASK = 0, 1
LFE_TOP_IS_EDGE, LFE_BOTTOM_IS_EDGE = 1, 2
LFE_PEER_ROWS = 8  # rows lfe_extract_rows_peer reads from each neighbour
LFE_OPT_KERNEL, LFE_OPT_TILE_W, LFE_OPT_TILE_H, LFE_OPT_HOST_STRIP_ROWS = 1, 2, 3, 4
LFE_KERNEL_AUTO, LFE_KERNEL_STAGED, LFE_KERNEL_FUSED = 0, 1, 2
LFE_OPT_LOG_UNIT = 5
LFE_LOG_AUTO, LFE_LOG_CUDA_CORES, LFE_LOG_TENSOR_CORES = 0, 1, 2  # fused kernel LoG unit (lfe.h)
LFE_ADAPT_ZC, LFE_ADAPT_STD = 1, 2

_STATUS = {0: "LFE_OK", 1: "LFE_EINVAL", 2: "LFE_EUNSUPPORTED", 3: "LFE_ENOMEM",
           4: "LFE_ENODEV", 5: "LFE_ECUDA", 6: "LFE_ERANGE"}


class LfeError(RuntimeError):
    def __init__(self, status: int, where: str, detail: str):
        self.status = status
        super().__init__(f"{where}: {_STATUS.get(status, status)}: {detail}")


class lfe_params(ctypes.Structure):
    _fields_ = [
        ("abi_size", ctypes.c_uint32),
        ("bit_depth", ctypes.c_int32),
        ("sigma", ctypes.c_double * 2),
        ("sigma_is_variance", ctypes.c_int32),
        ("log_size", ctypes.c_int32 * 2),
        ("adaptive", ctypes.c_int32),
        ("zc_threshold", ctypes.c_double * 2),
        ("std_source", ctypes.c_int32),
        ("std_window", ctypes.c_int32),
        ("std_threshold", ctypes.c_double * 2),
        ("std3_threshold", ctypes.c_double * 2),
        ("hybrid_median", ctypes.c_int32),
        ("median_window", ctypes.c_int32),
        ("out_mode", ctypes.c_int32),
        ("median_window2", ctypes.c_int32),
        ("mask_mode", ctypes.c_int32),
        ("reserved1", ctypes.c_int32),
    ]


assert ctypes.sizeof(lfe_params) == 120


class lfe_stats(ctypes.Structure):
    """Exact global sums for the adaptive thresholds (include/lfe.h; additive)."""
    _fields_ = [
        ("n", ctypes.c_int64),
        ("r_sum", ctypes.c_int64 * 2),
        ("r_sq_hi", ctypes.c_int64 * 2),
        ("r_sq_lo", ctypes.c_int64 * 2),
        ("i_sum", ctypes.c_int64),
        ("i_sq", ctypes.c_int64),
    ]


assert ctypes.sizeof(lfe_stats) == 72

_lib = None

# every symbol include/lfe.h declares (the CPU test checks the .so exports them)
EXPORTS = ["lfe_params_default", "lfe_create", "lfe_extract", "lfe_extract_rows", "lfe_extract_host",
           "lfe_halo", "lfe_get_mask", "lfe_last_async_error", "lfe_set_option", "lfe_launch_count",
           "lfe_destroy", "lfe_strerror", "lfe_last_message", "lfe_abi_version", "lfe_stats_rows",
           "lfe_set_stats", "lfe_get_thresholds", "lfe_extract_bands", "lfe_extract_rows_peer", "lfe_signal",
           "lfe_ipc_export", "lfe_ipc_open", "lfe_ipc_close", "lfe_set_stats_device"]
# include/lfe_test.h, exported by the separate liblfe_test.so
TEST_EXPORTS = ["lfe_test_mask", "lfe_test_validate", "lfe_test_response", "lfe_test_extract_r", "lfe_test_extract_e",
                "lfe_test_resolve"]
_test_lib = None


def load():
    """Load liblfe.so (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"liblfe.so not built ({LIB_PATH}); run __graft_entry__.build()")
    L = ctypes.CDLL(LIB_PATH)
    P, I32, I64, U32 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_uint32
    st = ctypes.c_int
    L.lfe_params_default.argtypes = [ctypes.POINTER(lfe_params)]
    L.lfe_params_default.restype = None
    L.lfe_create.argtypes = [ctypes.POINTER(lfe_params), ctypes.POINTER(P)]
    L.lfe_create.restype = st
    L.lfe_extract.argtypes = [P, P, I64, I32, I32, P, I64, P]
    L.lfe_extract.restype = st
    L.lfe_extract_rows.argtypes = [P, P, I64, I32, I32, I32, I32, U32, P, I64, P]
    L.lfe_extract_rows.restype = st
    L.lfe_extract_host.argtypes = [P, P, I64, I32, I32, P, I64]
    L.lfe_extract_host.restype = st
    L.lfe_halo.argtypes = [P]
    L.lfe_halo.restype = I32
    L.lfe_get_mask.argtypes = [P, I32, P, P, P, P]
    L.lfe_get_mask.restype = st
    L.lfe_last_async_error.argtypes = [P, P]
    L.lfe_last_async_error.restype = st
    L.lfe_set_option.argtypes = [P, I32, I64]
    L.lfe_set_option.restype = st
    L.lfe_launch_count.argtypes = [P]
    L.lfe_launch_count.restype = I64
    L.lfe_destroy.argtypes = [P]
    L.lfe_destroy.restype = None
    L.lfe_strerror.argtypes = [st]
    L.lfe_strerror.restype = ctypes.c_char_p
    L.lfe_last_message.argtypes = []
    L.lfe_last_message.restype = ctypes.c_char_p
    L.lfe_abi_version.argtypes = []
    L.lfe_abi_version.restype = I32
    L.lfe_extract_bands.argtypes = [P, P, I64, I64, I32, I32, I32, P, I64, I64, P]
    L.lfe_extract_bands.restype = st
    L.lfe_stats_rows.argtypes = [P, P, I64, I32, I32, I32, I32, U32, P, P]
    L.lfe_stats_rows.restype = st
    L.lfe_set_stats.argtypes = [P, ctypes.POINTER(lfe_stats)]
    L.lfe_set_stats.restype = st
    L.lfe_get_thresholds.argtypes = [P, P, P, P]
    L.lfe_get_thresholds.restype = st
    if hasattr(L, "lfe_extract_rows_peer"):  # (absent only in older builds loaded for A/B timing)
        L.lfe_extract_rows_peer.argtypes = [P, P, I64, I32, I32, P, I64, P, I64, U32, P, P, ctypes.c_uint64, P,
                                            I64, P]
        L.lfe_extract_rows_peer.restype = st
        L.lfe_signal.argtypes = [P, ctypes.c_uint64, P]
        L.lfe_signal.restype = st
        L.lfe_ipc_export.argtypes = [P, ctypes.c_char_p, ctypes.POINTER(I64)]
        L.lfe_ipc_export.restype = st
        L.lfe_ipc_open.argtypes = [ctypes.c_char_p, I64, ctypes.POINTER(P)]
        L.lfe_ipc_open.restype = st
        L.lfe_ipc_close.argtypes = [P, I64]
        L.lfe_ipc_close.restype = st
    if hasattr(L, "lfe_set_stats_device"):
        L.lfe_set_stats_device.argtypes = [P, P, P]
        L.lfe_set_stats_device.restype = st
    _lib = L
    return L


def load_test():
    """Load liblfe_test.so, the test-only entry points (include/lfe_test.h); it
    resolves the host core from the liblfe.so next to it."""
    global _test_lib
    if _test_lib is not None:
        return _test_lib
    load()
    if not os.path.exists(TEST_LIB_PATH):
        raise RuntimeError(f"liblfe_test.so not built ({TEST_LIB_PATH}); run __graft_entry__.build()")
    T = ctypes.CDLL(TEST_LIB_PATH)
    P, I32, I64 = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64
    st = ctypes.c_int
    T.lfe_test_mask.argtypes = [ctypes.c_double, I32, I32, P, P]
    T.lfe_test_mask.restype = st
    T.lfe_test_validate.argtypes = [ctypes.POINTER(lfe_params)]
    T.lfe_test_validate.restype = st
    T.lfe_test_response.argtypes = [P, P, I64, I32, I32, I32, P, P]
    T.lfe_test_response.restype = st
    T.lfe_test_extract_r.argtypes = [P, P, I64, I32, I32, P, I64, P]
    T.lfe_test_extract_r.restype = st
    T.lfe_test_extract_e.argtypes = [P, P, I64, I32, I32, P, I64, P]
    T.lfe_test_extract_e.restype = st
    T.lfe_test_resolve.argtypes = [P, ctypes.POINTER(lfe_stats), P]
    T.lfe_test_resolve.restype = st
    _test_lib = T
    return T


def _check(status: int, where: str):
    if status != LFE_OK:
        raise LfeError(status, where, load().lfe_last_message().decode())


# ------------------------------------------------------------ C names ----
def lfe_params_default() -> lfe_params:
    p = lfe_params()
    load().lfe_params_default(ctypes.byref(p))
    return p


def lfe_create(p: lfe_params) -> ctypes.c_void_p:
    h = ctypes.c_void_p()
    _check(load().lfe_create(ctypes.byref(p), ctypes.byref(h)), "lfe_create")
    return h


def lfe_extract(ctx, d_in: int, in_pitch: int, width: int, height: int, d_out: int, out_pitch: int,
                stream: int = 0):
    _check(load().lfe_extract(ctx, d_in, in_pitch, width, height, d_out, out_pitch, stream), "lfe_extract")


def lfe_extract_rows(ctx, d_in_row0: int, in_pitch: int, width: int, rows: int, halo_above: int,
                     halo_below: int, edge_flags: int, d_out_row0: int, out_pitch: int, stream: int = 0):
    _check(load().lfe_extract_rows(ctx, d_in_row0, in_pitch, width, rows, halo_above, halo_below,
                                   edge_flags, d_out_row0, out_pitch, stream), "lfe_extract_rows")


def lfe_extract_rows_peer(ctx, d_in_row0: int, in_pitch: int, width: int, rows: int, d_above: int, above_pitch: int,
                          d_below: int, below_pitch: int, edge_flags: int, wait_above: int, wait_below: int,
                          wait_value: int, d_out_row0: int, out_pitch: int, stream: int = 0):
    _check(load().lfe_extract_rows_peer(ctx, d_in_row0, in_pitch, width, rows, d_above or None, above_pitch,
                                        d_below or None, below_pitch, edge_flags, wait_above or None,
                                        wait_below or None, wait_value, d_out_row0, out_pitch, stream),
           "lfe_extract_rows_peer")


def lfe_signal(d_flag: int, value: int, stream: int = 0):
    _check(load().lfe_signal(d_flag, value, stream), "lfe_signal")


def lfe_ipc_export(d_ptr: int):
    """-> (64-byte handle, offset of d_ptr in its allocation)"""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64()
    _check(load().lfe_ipc_export(d_ptr, h, ctypes.byref(off)), "lfe_ipc_export")
    return h.raw, off.value


def lfe_ipc_open(handle: bytes, offset: int) -> int:
    p = ctypes.c_void_p()
    _check(load().lfe_ipc_open(handle, offset, ctypes.byref(p)), "lfe_ipc_open")
    return p.value


def lfe_ipc_close(d_ptr: int, offset: int):
    _check(load().lfe_ipc_close(d_ptr, offset), "lfe_ipc_close")


def lfe_extract_host(ctx, h_in: int, in_pitch: int, width: int, height: int, h_out: int, out_pitch: int):
    _check(load().lfe_extract_host(ctx, h_in, in_pitch, width, height, h_out, out_pitch), "lfe_extract_host")


def lfe_extract_bands(ctx, d_in: int, in_pitch: int, in_band_stride: int, width: int, height: int, bands: int,
                      d_out: int, out_pitch: int, out_band_stride: int, stream: int = 0):
    _check(load().lfe_extract_bands(ctx, d_in, in_pitch, in_band_stride, width, height, bands, d_out, out_pitch,
                                    out_band_stride, stream), "lfe_extract_bands")


def lfe_stats_rows(ctx, d_in_row0: int, in_pitch: int, width: int, rows: int, halo_above: int,
                   halo_below: int, edge_flags: int, d_stats: int, stream: int = 0):
    _check(load().lfe_stats_rows(ctx, d_in_row0, in_pitch, width, rows, halo_above, halo_below, edge_flags,
                                 d_stats, stream), "lfe_stats_rows")


def lfe_set_stats(ctx, stats: lfe_stats | None):
    _check(load().lfe_set_stats(ctx, ctypes.byref(stats) if stats is not None else None), "lfe_set_stats")


def lfe_get_thresholds(ctx):
    """(zc_t[2], std_T[2], std3_T[2]) in force."""
    z = (ctypes.c_int64 * 2)()
    t = (ctypes.c_double * 2)()
    t3 = (ctypes.c_double * 2)()
    _check(load().lfe_get_thresholds(ctx, z, t, t3), "lfe_get_thresholds")
    return tuple(z), tuple(t), tuple(t3)


def lfe_halo(ctx) -> int:
    return int(load().lfe_halo(ctx))


def lfe_get_mask(ctx, branch: int):
    coeffs = (ctypes.c_int32 * 81)()
    n, F, t = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int64()
    _check(load().lfe_get_mask(ctx, branch, coeffs, ctypes.byref(n), ctypes.byref(F), ctypes.byref(t)),
           "lfe_get_mask")
    q = np.array(coeffs[: n.value * n.value], np.int32).reshape(n.value, n.value)
    return q, F.value, t.value


def lfe_last_async_error(ctx, stream: int = 0) -> int:
    return int(load().lfe_last_async_error(ctx, stream))


def lfe_set_option(ctx, key: int, value: int):
    _check(load().lfe_set_option(ctx, key, value), "lfe_set_option")


def lfe_launch_count(ctx) -> int:
    return int(load().lfe_launch_count(ctx))


def lfe_destroy(ctx):
    load().lfe_destroy(ctx)


def lfe_strerror(status: int) -> str:
    return load().lfe_strerror(status).decode()


def lfe_abi_version() -> int:
    return int(load().lfe_abi_version())


def lfe_test_mask(sigma: float, n: int, bit_depth: int):
    """Host-side mask synthesis of the library (include/lfe_test.h)."""
    q = np.zeros(n * n, np.int32)
    F = ctypes.c_int32()
    _check(load_test().lfe_test_mask(float(sigma), n, bit_depth, q.ctypes.data, ctypes.byref(F)), "lfe_test_mask")
    return q.reshape(n, n), F.value


def lfe_test_validate(p: lfe_params) -> int:
    return int(load_test().lfe_test_validate(ctypes.byref(p)))


# ------------------------------------------------------ convenience ----
@dataclass
class Params:
    """Python view of lfe_params (defaults = lfe_params_default)."""
    bit_depth: int = 8
    sigma: tuple = (0.5, 20.0)
    sigma_is_variance: bool = False
    log_size: tuple = (5, 5)
    zc_threshold: tuple = (0.0, 0.0)
    std_source: int = LFE_STD_ZC
    std_window: int = 5
    std_threshold: tuple = (0.3, 0.3)
    std3_threshold: tuple = (-1.0, -1.0)
    hybrid_median: bool = True
    median_window: int = 5
    out_mode: int = LFE_OUT_EXTRACT
    median_window2: int = 0  # second hybrid-median level (water-body pipeline)
    adaptive: int = 0        # LFE_ADAPT_* (readings R21, R22)
    mask_mode: int = LFE_MASK_INT  # LFE_MASK_F32: float masks, tolerance contract (R23)

    def to_c(self) -> lfe_params:
        p = lfe_params()
        p.abi_size = ctypes.sizeof(lfe_params)
        p.bit_depth = self.bit_depth
        p.sigma[0], p.sigma[1] = self.sigma
        p.sigma_is_variance = int(bool(self.sigma_is_variance))
        p.log_size[0], p.log_size[1] = self.log_size
        p.zc_threshold[0], p.zc_threshold[1] = self.zc_threshold
        p.std_source = self.std_source
        p.std_window = self.std_window
        p.std_threshold[0], p.std_threshold[1] = self.std_threshold
        p.std3_threshold[0], p.std3_threshold[1] = self.std3_threshold
        p.hybrid_median = int(bool(self.hybrid_median))
        p.median_window = self.median_window
        p.out_mode = self.out_mode
        p.median_window2 = self.median_window2
        p.adaptive = self.adaptive
        p.mask_mode = self.mask_mode
        return p


def _in_dtype(bit_depth):
    return np.uint8 if bit_depth <= 8 else np.uint16


class Context:
    """One lfe_ctx: masks synthesised once, then any number of extractions."""

    def __init__(self, params: Params | None = None, **kw):
        self.params = params if params is not None else Params(**kw)
        self.handle = lfe_create(self.params.to_c())

    # -- metadata
    @property
    def halo(self) -> int:
        return lfe_halo(self.handle)

    def mask(self, branch: int):
        return lfe_get_mask(self.handle, branch)

    def set_option(self, key: int, value: int):
        lfe_set_option(self.handle, key, value)

    @property
    def launches(self) -> int:
        return lfe_launch_count(self.handle)

    def in_dtype(self):
        return _in_dtype(self.params.bit_depth)

    def out_dtype(self):
        return np.uint8 if self.params.out_mode == LFE_OUT_MASK else self.in_dtype()

    # -- device (torch) entry points
    @staticmethod
    def _torch_img(t, name):
        import torch
        if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
            raise TypeError(f"{name} must be a CUDA torch tensor")
        if t.dim() != 2 or t.stride(1) != 1:
            raise ValueError(f"{name} must be 2-D with unit column stride")
        return t.data_ptr(), t.stride(0) * t.element_size()

    @staticmethod
    def _stream(stream):
        import torch
        if stream is None:
            return torch.cuda.current_stream().cuda_stream
        return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)

    def _check_dtype(self, t_in, t_out):
        import torch
        tin = torch.uint8 if self.params.bit_depth <= 8 else torch.uint16
        tout = torch.uint8 if self.params.out_mode == LFE_OUT_MASK else tin
        if t_in.dtype != tin or t_out.dtype != tout:
            raise TypeError(f"dtypes must be {tin} -> {tout}")

    def extract(self, t_in, t_out=None, stream=None):
        """Whole-image extraction of a 2-D CUDA tensor; returns the output tensor."""
        import torch
        if t_out is None:
            tout = torch.uint8 if self.params.out_mode == LFE_OUT_MASK else t_in.dtype
            t_out = torch.empty(t_in.shape, dtype=tout, device=t_in.device)
        self._check_dtype(t_in, t_out)
        if t_in.shape != t_out.shape:
            raise ValueError("shape mismatch")
        pi, pin = self._torch_img(t_in, "input")
        po, pout = self._torch_img(t_out, "output")
        H, W = t_in.shape
        lfe_extract(self.handle, pi, pin, W, H, po, pout, self._stream(stream))
        return t_out

    def extract_bands(self, t_in, t_out=None, stream=None):
        """All bands of a [B, H, W] CUDA tensor in one launch (lfe_extract_bands)."""
        import torch
        if t_in.dim() != 3 or t_in.stride(2) != 1:
            raise ValueError("input must be [bands, H, W] with unit column stride")
        if t_out is None:
            tout = torch.uint8 if self.params.out_mode == LFE_OUT_MASK else t_in.dtype
            t_out = torch.empty(t_in.shape, dtype=tout, device=t_in.device)
        self._check_dtype(t_in, t_out)
        B, H, W = t_in.shape
        e_in, e_out = t_in.element_size(), t_out.element_size()
        lfe_extract_bands(self.handle, t_in.data_ptr(), t_in.stride(1) * e_in, t_in.stride(0) * e_in, W, H, B,
                          t_out.data_ptr(), t_out.stride(1) * e_out, t_out.stride(0) * e_out, self._stream(stream))
        return t_out

    def extract_rows_peer(self, t_own, t_out, above=None, below=None, wait_above=None, wait_below=None,
                          wait_value: int = 0, edge_flags: int | None = None, stream=None):
        """lfe_extract_rows_peer on torch views: t_own = the strip's owned rows,
        above / below = views whose first row is the first halo row above / below
        the strip (None = that side is the image edge), wait_* = int64 flag
        tensors (or raw pointers) the kernel waits on."""
        self._check_dtype(t_own, t_out)
        W = t_own.shape[1]
        e_in, e_out = t_own.element_size(), t_out.element_size()

        def ptr(t):
            return 0 if t is None else (t if isinstance(t, int) else t.data_ptr())

        def pitch(t):
            return 0 if t is None or isinstance(t, int) else t.stride(0) * e_in

        if edge_flags is None:
            edge_flags = (LFE_TOP_IS_EDGE if above is None else 0) | (LFE_BOTTOM_IS_EDGE if below is None else 0)
        lfe_extract_rows_peer(self.handle, t_own.data_ptr(), t_own.stride(0) * e_in, W, t_own.shape[0],
                              ptr(above), pitch(above), ptr(below), pitch(below), edge_flags, ptr(wait_above),
                              ptr(wait_below), wait_value, t_out.data_ptr(), t_out.stride(0) * e_out,
                              self._stream(stream))
        return t_out

    def extract_rows(self, t_in_full, row0: int, rows: int, halo_above: int, halo_below: int,
                     edge_flags: int, t_out, out_row0: int = 0, stream=None):
        """Strip entry point: t_in_full holds rows [row0-halo_above, row0+rows+halo_below)."""
        pi, pin = self._torch_img(t_in_full, "input")
        po, pout = self._torch_img(t_out, "output")
        self._check_dtype(t_in_full, t_out)
        W = t_in_full.shape[1]
        lfe_extract_rows(self.handle, pi + row0 * pin, pin, W, rows, halo_above, halo_below, edge_flags,
                         po + out_row0 * pout, pout, self._stream(stream))
        return t_out

    def stats_rows(self, t_in_full, row0: int, rows: int, halo_above: int, halo_below: int,
                   edge_flags: int, t_stats, stream=None):
        """Adds the owned rows' exact sums to t_stats (a CUDA int64 tensor of 9)."""
        import torch
        pi, pin = self._torch_img(t_in_full, "input")
        if t_stats.dtype != torch.int64 or t_stats.numel() != 9 or t_stats.device.type != "cuda":
            raise TypeError("t_stats must be a CUDA int64 tensor of 9 elements")
        W = t_in_full.shape[1]
        lfe_stats_rows(self.handle, pi + row0 * pin, pin, W, rows, halo_above, halo_below, edge_flags,
                       t_stats.data_ptr(), self._stream(stream))
        return t_stats

    @staticmethod
    def stats_from(values) -> lfe_stats:
        """lfe_stats from 9 int64 values in field order."""
        v = [int(x) for x in values]
        s = lfe_stats()
        s.n = v[0]
        s.r_sum[0], s.r_sum[1] = v[1], v[2]
        s.r_sq_hi[0], s.r_sq_hi[1] = v[3], v[4]
        s.r_sq_lo[0], s.r_sq_lo[1] = v[5], v[6]
        s.i_sum, s.i_sq = v[7], v[8]
        return s

    def set_stats(self, stats):
        """Whole-image statistics (an lfe_stats, or 9 int64 values) -> thresholds."""
        if stats is not None and not isinstance(stats, lfe_stats):
            stats = self.stats_from(stats)
        lfe_set_stats(self.handle, stats)

    def thresholds(self):
        return lfe_get_thresholds(self.handle)

    def set_stats_device(self, t_stats, stream=None):
        """lfe_set_stats_device: resolve the thresholds on the device from a CUDA
        int64 tensor of the 9 lfe_stats values (no host round trip)."""
        _check(load().lfe_set_stats_device(self.handle, t_stats.data_ptr(), self._stream(stream)),
               "lfe_set_stats_device")

    def test_resolve(self, values):
        """lfe_test_resolve: the device resolution of host statistics -> (t_0, t_1)."""
        z = (ctypes.c_int64 * 2)()
        s = values if isinstance(values, lfe_stats) else self.stats_from(values)
        _check(load_test().lfe_test_resolve(self.handle, ctypes.byref(s), z), "lfe_test_resolve")
        return z[0], z[1]

    def test_response(self, t_in, branch: int, stream=None):
        """lfe_test_response: branch's LoG response of a whole device image as the
        general kernel computes it (int32, or float32 in F32 mode)."""
        import torch
        pi, pin = self._torch_img(t_in, "input")
        H, W = t_in.shape
        dt = torch.float32 if self.params.mask_mode == LFE_MASK_F32 else torch.int32
        out = torch.empty((H, W), dtype=dt, device=t_in.device)
        _check(load_test().lfe_test_response(self.handle, pi, pin, W, H, branch, out.data_ptr(), self._stream(stream)),
               "lfe_test_response")
        return out

    def test_extract_r(self, t_in, t_out, stream=None):
        """lfe_test_extract_r: the fused kernel on injected responses (include/lfe_test.h)."""
        pi, pin = self._torch_img(t_in, "input")
        po, pout = self._torch_img(t_out, "output")
        H, W = t_in.shape
        _check(load_test().lfe_test_extract_r(self.handle, pi, pin, W, H, po, pout, self._stream(stream)),
               "lfe_test_extract_r")
        return t_out

    def test_extract_e(self, t_in, t_out, stream=None):
        """lfe_test_extract_e: the fused kernel's hybrid-median stages on E = the input
        (include/lfe_test.h)."""
        pi, pin = self._torch_img(t_in, "input")
        po, pout = self._torch_img(t_out, "output")
        H, W = t_in.shape
        _check(load_test().lfe_test_extract_e(self.handle, pi, pin, W, H, po, pout, self._stream(stream)),
               "lfe_test_extract_e")
        return t_out

    def last_async_error(self, stream=None) -> int:
        return lfe_last_async_error(self.handle, self._stream(stream))

    def check(self, stream=None):
        _check(self.last_async_error(stream), "lfe_last_async_error")

    # -- host entry point
    def extract_host(self, a_in: np.ndarray, a_out: np.ndarray | None = None) -> np.ndarray:
        """End to end on host memory (H2D -> kernel -> D2H inside liblfe)."""
        if a_in.ndim != 2 or a_in.strides[1] != a_in.itemsize:
            raise ValueError("input must be 2-D with unit column stride")
        if a_in.dtype != self.in_dtype():
            raise TypeError(f"input dtype must be {np.dtype(self.in_dtype())}")
        if a_out is None:
            a_out = np.empty(a_in.shape, self.out_dtype())
        if a_out.dtype != self.out_dtype() or a_out.shape != a_in.shape:
            raise TypeError("bad output array")
        H, W = a_in.shape
        lfe_extract_host(self.handle, a_in.ctypes.data, a_in.strides[0], W, H, a_out.ctypes.data,
                         a_out.strides[0])
        return a_out

    def extract_host_ptr(self, p_in: int, in_pitch: int, W: int, H: int, p_out: int, out_pitch: int):
        lfe_extract_host(self.handle, p_in, in_pitch, W, H, p_out, out_pitch)

    def close(self):
        if self.handle:
            lfe_destroy(self.handle)
            self.handle = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
