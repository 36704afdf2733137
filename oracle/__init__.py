"""CPU oracle for the arXiv 1304.3992 hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
and ``--impl reference`` legs may import this package.  The product path
(``paper_1304_3992_b200``) never imports it and shares no code with it.

Thin ctypes wrapper over ``lfe_oracle.c`` (plain C, int64/double, every stage
materialised in the order of PAPER.md:94, Sec. 4.1).  Each wrapper names the
passage its C function follows; see that file for the step-by-step code and
DESIGN.md "Readings" for R1..R20.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "lfe_oracle.c")
_LIB = os.path.join(_HERE, "liblfe_oracle.so")

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, OpenMP over rows, no intrinsics)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(
            ["gcc", "-O2", "-std=c11", "-fopenmp", "-fPIC", "-shared", _SRC, "-o", tmp, "-lm"]
        )
        os.replace(tmp, _LIB)
    return _LIB


class _Params(ctypes.Structure):
    _fields_ = [
        ("bit_depth", ctypes.c_int32),
        ("sigma_is_variance", ctypes.c_int32),
        ("sigma", ctypes.c_double * 2),
        ("log_size", ctypes.c_int32 * 2),
        ("zc_threshold", ctypes.c_double * 2),
        ("std_source", ctypes.c_int32),
        ("std_window", ctypes.c_int32),
        ("std_threshold", ctypes.c_double * 2),
        ("std3_threshold", ctypes.c_double * 2),
        ("hybrid_median", ctypes.c_int32),
        ("median_window", ctypes.c_int32),
        ("out_mode", ctypes.c_int32),
        ("median_window2", ctypes.c_int32),
        ("adaptive", ctypes.c_int32),
        ("mask_mode", ctypes.c_int32),
    ]


def lib():
    global _lib
    if _lib is None:
        # LFE_ORACLE_LIB: an instrumented build of the same source (ASan/UBSan runs,
        # tests/test_sanitizers.py) instead of the default one
        path = os.environ.get("LFE_ORACLE_LIB")
        if not path:
            build()
            path = _LIB
        L = ctypes.CDLL(path)
        P = ctypes.c_void_p
        L.lfo_set_threads.argtypes = [ctypes.c_int]
        L.lfo_get_threads.restype = ctypes.c_int
        L.lfo_log_raw.argtypes = [ctypes.c_double, ctypes.c_int, P]
        L.lfo_log_dc.argtypes = [ctypes.c_double, ctypes.c_int, P]
        L.lfo_mask_int.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_int, P, P]
        L.lfo_zc_threshold_int.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_int]
        L.lfo_zc_threshold_int.restype = ctypes.c_int64
        L.lfo_log_response.argtypes = [P, ctypes.c_int, ctypes.c_int, P, ctypes.c_int, P]
        L.lfo_zero_crossing.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int64, P]
        L.lfo_sample_std.argtypes = [P, ctypes.c_int]
        L.lfo_sample_std.restype = ctypes.c_double
        L.lfo_std_gate.argtypes = [P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                   ctypes.c_double, ctypes.c_double, P]
        L.lfo_merge.argtypes = [P, P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        L.lfo_hybrid_median.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_int, P]
        L.lfo_run.argtypes = [ctypes.POINTER(_Params), P, ctypes.c_int, ctypes.c_int, P,
                              P, P, P, P, P, P, P]
        L.lfo_run.restype = ctypes.c_int
        L.lfo_mask_f32.argtypes = [ctypes.c_double, ctypes.c_int, P, P]
        L.lfo_log_response_f.argtypes = [P, ctypes.c_int, ctypes.c_int, P, ctypes.c_int, ctypes.c_double, P]
        L.lfo_zero_crossing_f.argtypes = [P, ctypes.c_int, ctypes.c_int, ctypes.c_double, P]
        L.lfo_std_gate_resp_int.argtypes = [P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                            ctypes.c_double, ctypes.c_int, P]
        L.lfo_std_gate_resp_f.argtypes = [P, P, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_double,
                                          ctypes.c_double, ctypes.c_int, P]
        L.lfo_global_std_parts.argtypes = [ctypes.c_int64, ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint64,
                                           ctypes.c_uint64]
        L.lfo_global_std_parts.restype = ctypes.c_double
        L.lfo_std_of_response.argtypes = [P, ctypes.c_size_t]
        L.lfo_std_of_response.restype = ctypes.c_double
        L.lfo_std_of_intensity.argtypes = [P, ctypes.c_size_t]
        L.lfo_std_of_intensity.restype = ctypes.c_double
        L.lfo_adaptive_zc_threshold.argtypes = [ctypes.c_double, ctypes.c_double]
        L.lfo_adaptive_zc_threshold.restype = ctypes.c_int64
        _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def set_threads(n: int) -> None:
    lib().lfo_set_threads(int(n))


def get_threads() -> int:
    return int(lib().lfo_get_threads())


# ---------------------------------------------------------------- masks ----
def log_raw(sigma: float, n: int) -> np.ndarray:
    """Eq. 1 sampled at integer offsets; [y, x] indexing."""
    out = np.empty((n, n), np.float64)
    if lib().lfo_log_raw(float(sigma), int(n), _ptr(out)) != 0:
        raise ValueError("bad sigma/size")
    return out


def log_dc(sigma: float, n: int) -> np.ndarray:
    """Eq. 1 minus its mean (reading R2)."""
    out = np.empty((n, n), np.float64)
    if lib().lfo_log_dc(float(sigma), int(n), _ptr(out)) != 0:
        raise ValueError("bad sigma/size")
    return out


def mask_int(sigma: float, n: int, bit_depth: int):
    """Integer mask and its shift F (reading R3). Returns (q[n,n] int32, F)."""
    q = np.empty((n, n), np.int32)
    F = ctypes.c_int(0)
    if lib().lfo_mask_int(float(sigma), int(n), int(bit_depth), _ptr(q), ctypes.byref(F)) != 0:
        raise ValueError("no admissible quantisation")
    return q, F.value


def zc_threshold_int(thr: float, F: int, bit_depth: int) -> int:
    return int(lib().lfo_zc_threshold_int(float(thr), int(F), int(bit_depth)))


# --------------------------------------------------------------- stages ----
def log_response(I: np.ndarray, q: np.ndarray) -> np.ndarray:
    """mask applied on each pixel's n x n neighbourhood (replicate pad)."""
    I = np.ascontiguousarray(I, dtype=np.uint16)
    q = np.ascontiguousarray(q, dtype=np.int32)
    H, W = I.shape
    r = np.empty((H, W), np.int64)
    lib().lfo_log_response(_ptr(I), W, H, _ptr(q), q.shape[0], _ptr(r))
    return r


def zero_crossing(r: np.ndarray, t: int = 0) -> np.ndarray:
    """PAPER.md:60 (Sec. 3.2) rule R*; r int64 [H, W]; returns uint8 0/1."""
    r = np.ascontiguousarray(r, dtype=np.int64)
    H, W = r.shape
    Z = np.empty((H, W), np.uint8)
    lib().lfo_zero_crossing(_ptr(r), W, H, int(t), _ptr(Z))
    return Z


def sample_std(a) -> float:
    """Eq. 2 literally."""
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64).ravel())
    return float(lib().lfo_sample_std(_ptr(a), a.size))


def std_gate(src: np.ndarray, Z: np.ndarray, w: int, T: float, T3: float = -1.0) -> np.ndarray:
    """PAPER.md:94 std gate over a w x w window (+ optional 3x3 re-check)."""
    src = np.ascontiguousarray(src, dtype=np.uint16)
    Z = np.ascontiguousarray(Z, dtype=np.uint8)
    H, W = Z.shape
    keep = np.empty((H, W), np.uint8)
    lib().lfo_std_gate(_ptr(src), _ptr(Z), W, H, int(w), float(T), float(T3), _ptr(keep))
    return keep


def merge(k0, k1, I, out_mode: int = 0) -> np.ndarray:
    k0 = np.ascontiguousarray(k0, dtype=np.uint8)
    k1 = np.ascontiguousarray(k1, dtype=np.uint8)
    I = np.ascontiguousarray(I, dtype=np.uint16)
    H, W = I.shape
    E = np.empty((H, W), np.uint16)
    lib().lfo_merge(_ptr(k0), _ptr(k1), _ptr(I), W, H, int(out_mode), _ptr(E))
    return E


def hybrid_median(E: np.ndarray, m: int = 5) -> np.ndarray:
    """PAPER.md:76 (Sec. 3.4): med3(median(+ group), median(x group), centre)."""
    E = np.ascontiguousarray(E, dtype=np.uint16)
    H, W = E.shape
    out = np.empty((H, W), np.uint16)
    lib().lfo_hybrid_median(_ptr(E), W, H, int(m), _ptr(out))
    return out


# ------------------------------------------------------- F32 mode (R23) ----
def mask_f32(sigma: float, n: int):
    """(float32 mask = (float) L_dc, c = |L_dc(0,0)|)."""
    w = np.empty((n, n), np.float32)
    c = ctypes.c_double()
    if lib().lfo_mask_f32(float(sigma), int(n), _ptr(w), ctypes.byref(c)) != 0:
        raise ValueError("bad sigma/size")
    return w, c.value


def log_response_f(I: np.ndarray, w: np.ndarray, scale: float) -> np.ndarray:
    """Normalised float response r^ = (w * I) * scale, |r^| < 1e-4 snapped to 0."""
    I = np.ascontiguousarray(I, dtype=np.uint16)
    w = np.ascontiguousarray(w, dtype=np.float32)
    H, W = I.shape
    r = np.empty((H, W), np.float64)
    lib().lfo_log_response_f(_ptr(I), W, H, _ptr(w), w.shape[0], float(scale), _ptr(r))
    return r


def zero_crossing_f(r: np.ndarray, t: float = 0.0) -> np.ndarray:
    r = np.ascontiguousarray(r, dtype=np.float64)
    H, W = r.shape
    Z = np.empty((H, W), np.uint8)
    lib().lfo_zero_crossing_f(_ptr(r), W, H, float(t), _ptr(Z))
    return Z


def std_gate_response(r: np.ndarray, Z: np.ndarray, w: int, T: float, T3: float = -1.0, at_zc: bool = False):
    """R24: std over the signed response window (int64 r: exact;
    float r: double), gated to ZC pixels.  T in the response's own units."""
    Z = np.ascontiguousarray(Z, dtype=np.uint8)
    H, W = Z.shape
    keep = np.empty((H, W), np.uint8)
    if np.issubdtype(r.dtype, np.integer):
        r = np.ascontiguousarray(r, dtype=np.int64)
        lib().lfo_std_gate_resp_int(_ptr(r), _ptr(Z), W, H, int(w), float(T), float(T3), int(at_zc), _ptr(keep))
    else:
        r = np.ascontiguousarray(r, dtype=np.float64)
        lib().lfo_std_gate_resp_f(_ptr(r), _ptr(Z), W, H, int(w), float(T), float(T3), int(at_zc), _ptr(keep))
    return keep


# ------------------------------------------------- adaptive thresholds ----
def global_std(n: int, s1: int, s2: int) -> float:
    """R21: sqrt(n*S2 - S1^2) / n from exact integer sums (Python ints)."""
    m = (1 << 64) - 1
    s1u = s1 & ((1 << 128) - 1)
    return float(lib().lfo_global_std_parts(int(n), s1u >> 64, s1u & m, (s2 >> 64) & m, s2 & m))


def std_of_response(r: np.ndarray) -> float:
    """global (population) standard deviation of a LoG response."""
    r = np.ascontiguousarray(r, dtype=np.int64)
    return float(lib().lfo_std_of_response(_ptr(r), r.size))


def std_of_intensity(I: np.ndarray) -> float:
    """global (population) standard deviation of the band."""
    I = np.ascontiguousarray(I, dtype=np.uint16)
    return float(lib().lfo_std_of_intensity(_ptr(I), I.size))


def adaptive_zc_threshold(k: float, sigma_r: float) -> int:
    return int(lib().lfo_adaptive_zc_threshold(float(k), float(sigma_r)))


# ------------------------------------------------------------- pipeline ----
@dataclass
class Params:
    """Oracle-side parameter set (independent of include/lfe.h)."""
    bit_depth: int = 8
    sigma: tuple = (0.5, 20.0)
    sigma_is_variance: bool = False
    log_size: tuple = (5, 5)
    zc_threshold: tuple = (0.0, 0.0)
    std_source: int = 0
    std_window: int = 5
    std_threshold: tuple = (0.3, 0.3)
    std3_threshold: tuple = (-1.0, -1.0)
    hybrid_median: bool = True
    median_window: int = 5
    out_mode: int = 0
    median_window2: int = 0
    adaptive: int = 0  # bit 0: ZC gap k * sigma_r (R21); bit 1: std thresholds k * sigma_I (R22)
    mask_mode: int = 0  # 0 integer masks (R3); 1 float masks + normalised response (R23)

    def to_c(self) -> _Params:
        p = _Params()
        p.bit_depth = self.bit_depth
        p.sigma_is_variance = int(bool(self.sigma_is_variance))
        p.sigma[0], p.sigma[1] = self.sigma
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


@dataclass
class Result:
    out: np.ndarray
    r: list = field(default_factory=list)
    z: list = field(default_factory=list)
    keep: list = field(default_factory=list)
    E: np.ndarray | None = None


def run(I: np.ndarray, params: Params, intermediates: bool = False):
    """Whole pipeline (Fig. 1 + optional Sec. 3.4 hybrid median).

    Returns the output image (same dtype as I for extract mode, uint8 for the
    mask mode), or a Result with every intermediate if ``intermediates``.
    """
    src_dtype = I.dtype
    I16 = np.ascontiguousarray(I, dtype=np.uint16)
    H, W = I16.shape
    out = np.empty((H, W), np.uint16)
    if intermediates:
        r0, r1 = np.empty((H, W), np.int64), np.empty((H, W), np.int64)
        z0, z1, k0, k1 = (np.empty((H, W), np.uint8) for _ in range(4))
        E = np.empty((H, W), np.uint16)
    else:
        r0 = r1 = z0 = z1 = k0 = k1 = E = None
    cp = params.to_c()
    rc = lib().lfo_run(ctypes.byref(cp), _ptr(I16), W, H, _ptr(out), _ptr(r0), _ptr(r1),
                       _ptr(z0), _ptr(z1), _ptr(k0), _ptr(k1), _ptr(E))
    if rc == -3:
        raise ValueError("pixel value exceeds 2^bit_depth - 1")
    if rc != 0:
        raise ValueError(f"oracle run failed ({rc})")
    out_dtype = np.uint8 if params.out_mode == 1 else src_dtype
    out = out.astype(out_dtype)
    if not intermediates:
        return out
    if params.mask_mode == 1:  # F32 mode: the response buffers hold doubles (r^)
        r0, r1 = r0.view(np.float64), r1.view(np.float64)
    return Result(out=out, r=[r0, r1], z=[z0, z1], keep=[k0, k1], E=E)
