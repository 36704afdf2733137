#!/usr/bin/env python
"""Benchmark of the dual-LoG feature-extraction hot path (arXiv 1304.3992) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lfe|reference] [--config c1..c5]

A step = one pass of the whole hot path (LoG x2 -> zero crossing -> std gate ->
OR merge -> hybrid median) over one scene of the chosen BASELINE.json config,
resident in HBM.  The default (the metric line) is c3: 12000 x 12000 uint16
(10-bit), Cartosat-1-like synthetic PAN.  The other configs are per-scene
throughput lines (Table 6 reports every test image):
  c1  512^2 u8      one launch per step, replayed as a CUDA graph at N = 1
  c2  4096^2 u8
  c4  4 x 8192^2 u16 (12-bit) bands: all bands in one lfe_extract_bands launch;
      across GPUs the band-major rows are dealt out (plan_bands): whole bands need
      no collective, a band cut between two ranks gets a halo exchange
  c5  48000^2 u16 mosaic: value = device-resident strips; e2e = the scene streamed
      from pinned host memory through lfe_extract_host (H2D / kernel / D2H overlap)
At N > 1 (torchrun, one process per GPU) a scene is split into N row strips with
an NCCL halo exchange of the boundary rows (strong scaling: the scene is fixed).
After the timed steps the output of the last step is compared with the CPU
oracle ("parity": whole scene for c1-c4, 13 row bands for c5; every rank checks
its own rows).  --median2 3 adds the water pipeline's second median level
(PAPER.md:102); --adaptive k the adaptive ZC gap.  Rank 0 prints
one JSON line.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "megapixels/s per scene at 1/2/4/8 B200; achieved HBM GB/s fraction of peak"
UNIT = "Mpx/s"
FALLBACK_HBM_GBS = 6650.0  # /opt/skills/guides/B200_PROFILING.md fallback

# the fused kernel's sources: committed ncu numbers (profiles/issue.json, traffic.json)
# carry the hash of the sources they were captured from
FUSED_SOURCES = ["paper_1304_3992_b200/csrc/kernel_fused.cuh", "paper_1304_3992_b200/csrc/kernel_fused.cu"]


def fused_source_hash() -> str:
    h = hashlib.sha256()
    for f in FUSED_SOURCES:
        with open(os.path.join(ROOT, f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


# ---------------------------------------------------------------- configs ----
CFG = {
    "c1": dict(bit_depth=8, zc=0.02, H=512, W=512, bands=1,
               desc="c1: 512x512 uint8 synthetic panchromatic (steps, disks, lines + 1% salt-and-pepper)"),
    "c2": dict(bit_depth=8, zc=0.02, H=4096, W=4096, bands=1,
               desc="c2: 4096x4096 uint8 synthetic urban-like panchromatic tile"),
    "c3": dict(bit_depth=10, zc=0.02, H=12000, W=12000, bands=1,
               desc="c3: 12000x12000 uint16 (10-bit) synthetic Cartosat-1-like PAN scene"),
    "c4": dict(bit_depth=12, zc=0.01, H=8192, W=8192, bands=4,
               desc="c4: 4-band 8192x8192 uint16 (12-bit) synthetic AWiFS-like multispectral scene, per-band pipeline"),
    "c5": dict(bit_depth=10, zc=0.02, H=48000, W=48000, bands=1,
               desc="c5: 48000x48000 uint16 (10-bit) PAN mosaic of 4x4 c3-generator tiles"),
}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["lfe", "reference"], default="lfe")
    ap.add_argument("--config", choices=sorted(CFG), default="c3")
    ap.add_argument("--kernel", choices=["auto", "staged", "fused"], default="auto")
    ap.add_argument("--log-unit", choices=["auto", "cuda", "tensor"], default="auto",
                    help="fused kernel LoG: tensor cores where exact and worthwhile (auto), forced CUDA cores, "
                         "or tensor cores wherever exact (A/B)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true", help="do not report the oracle timing")
    ap.add_argument("--no-parity", action="store_true", help="skip the oracle parity check of the last step")
    ap.add_argument("--no-graph", action="store_true", help="c1/c2 at N=1: plain launches instead of graph replay")
    ap.add_argument("--halo", choices=["auto", "peer", "nccl"], default="auto",
                    help="N > 1 row strips: 'peer' = one launch per step reading the halo rows from the "
                         "neighbours' HBM (CUDA IPC, lfe_extract_rows_peer); 'nccl' = NCCL halo exchange with "
                         "the interior band overlapped; auto = peer (nccl for --adaptive)")
    ap.add_argument("--verify", action="store_true",
                    help="after timing, check every rank's owned output rows against a whole-scene "
                         "extraction on its own GPU (bit-exact); adds \"verify\" to the line")
    ap.add_argument("--size", type=int, default=0, help="c3 scene side / c4 band side override (tests / tuning)")
    ap.add_argument("--tile", type=str, default="", help="TWxTH override (tuning only)")
    ap.add_argument("--median2", type=int, default=0, choices=[0, 3, 5, 7],
                    help="second hybrid-median level (the water pipeline, PAPER.md:102); 0 = the metric config")
    ap.add_argument("--std", choices=["zc", "intensity"], default="zc",
                    help="image the Eq. 2 deviation is computed on (reading R10): the ZC image (the metric config) "
                         "or the intensity image (R10's alternative; T = 20 DN x 2^(b-10))")
    ap.add_argument("--adaptive", type=float, default=0.0,
                    help="k > 0: adaptive ZC gap t = ceil(k * sigma(r)) (SPEC.md:233, NEXT-2), with its "
                         "statistics pre-pass and all-reduce inside every step; 0 = the metric config")
    a = ap.parse_args()
    if a.size and a.config not in ("c3", "c4"):
        ap.error("--size applies to c3 and c4 only")
    if a.config in ("c4", "c5") and (a.adaptive or a.verify):
        ap.error("--adaptive / --verify are wired for the single-scene configs c1-c3 only")
    return a


def geometry(args):
    c = dict(CFG[args.config])
    if args.config in ("c3", "c4") and args.size:
        c["H"] = c["W"] = args.size
    return c


def workload_params(cfg, median2=0, adaptive=0.0, std="zc"):
    from paper_1304_3992_b200 import lfe
    # SURVEY.md 8(c) defaults for benchmark scenes: ZC gap 0.02 (normalised; 0.01 for the
    # 12-bit c4), std source = ZC image, 5x5 window, T = 0.3, hybrid median on, extract.
    zc = (adaptive, adaptive) if adaptive > 0 else (cfg["zc"], cfg["zc"])
    T = 0.3 if std == "zc" else 20.0 * 2.0 ** (cfg["bit_depth"] - 10)
    return lfe.Params(bit_depth=cfg["bit_depth"], sigma=(0.5, 20.0), log_size=(5, 5), zc_threshold=zc,
                      std_source=lfe.LFE_STD_ZC if std == "zc" else lfe.LFE_STD_INTENSITY, std_window=5,
                      std_threshold=(T, T),
                      std3_threshold=(-1.0, -1.0), hybrid_median=True, median_window=5,
                      out_mode=lfe.LFE_OUT_EXTRACT, median_window2=median2,
                      adaptive=lfe.LFE_ADAPT_ZC if adaptive > 0 else 0)


def oracle_params(p):
    import oracle
    return oracle.Params(bit_depth=p.bit_depth, sigma=p.sigma, log_size=p.log_size, zc_threshold=p.zc_threshold,
                         std_source=p.std_source, std_window=p.std_window, std_threshold=p.std_threshold,
                         std3_threshold=p.std3_threshold, hybrid_median=p.hybrid_median,
                         median_window=p.median_window, out_mode=p.out_mode, median_window2=p.median_window2,
                         adaptive=p.adaptive)


def halo_rows(p):
    """Rows of real input an output band needs above/below (north_star's halo)."""
    h = max(p.log_size) // 2 + 1 + p.std_window // 2
    if p.hybrid_median:
        h += p.median_window // 2 + p.median_window2 // 2
    return h


def elem(cfg):
    return 1 if cfg["bit_depth"] <= 8 else 2


def _backend_name():
    try:
        import torch.distributed as dist
        b = dist.get_backend() if dist.is_initialized() else "nccl"
    except Exception:
        b = "nccl"
    return "NCCL" if b == "nccl" else f"{b} (host-staged; ranks sharing a GPU: test hook, not a measurement)"


def log_unit_of(ctx, p, unit: str, units: int) -> str:
    """Which unit the fused kernel computes the two LoG responses on (the library's
    rule, kernel_fused.cu tc_exact): the tensor cores when exact there -- u16 input with
    b <= 12 and every mask coefficient an fp16 value -- else the CUDA cores."""
    import numpy as np
    qs = [ctx.mask(j)[0].astype(np.float64) for j in (0, 1)]
    hi = [np.float16(q).astype(np.float64) for q in qs]
    exact = all(np.all(h == q) for h, q in zip(hi, qs))
    split = all(np.all(np.float16(q - h).astype(np.float64) == q - h) for h, q in zip(hi, qs)) and \
        max(float(np.abs(h).sum() + np.abs(q - h).sum()) for h, q in zip(hi, qs)) * ((1 << p.bit_depth) - 1) < 2 ** 24
    tc = (8 < p.bit_depth <= 12 and exact) or (p.bit_depth <= 8 and split)
    tc = tc and (units >= 32 * 148 or unit == "tensor")  # the library's small-launch rule (kernel_fused.cu)
    if unit != "cuda" and tc and p.std_source == 0:
        return ("tensor cores (tcgen05.mma kind::f16 into TMEM; exact: the input bits as fp16 = v*2^-24"
                + ("; b = 12: v & 0x7FF and bit 11 as two K halves)" if p.bit_depth == 12 else
                   "; u8: weights as fp16(q) + remainder in two B matrices)" if p.bit_depth <= 8 else
                   ", fp16-exact integer masks)"))
    return "CUDA cores (exact-integer fp32 FFMA)"


def config_dict(name, cfg, world, p, graph=False, halo_mode=None, log_unit=None):
    hm = "5x5 hybrid median" + (f" + {p.median_window2}x{p.median_window2} second level" if p.median_window2 else "")
    zc = (f"ZC (adaptive gap {p.zc_threshold[0]} x global std of r, statistics pre-pass)" if p.adaptive
          else f"ZC (gap {p.zc_threshold[0]})")
    H, W, B, e = cfg["H"], cfg["W"], cfg["bands"], elem(cfg)
    in_bytes = B * H * W * e
    if world > 1:
        if B > 1:
            par = (f"bands dealt to {world} ranks (plan_bands; a band cut between two ranks gets a "
                   f"{halo_rows(p)}-row {_backend_name()} halo exchange)")
        elif halo_mode == "peer":
            par = (f"row strips x{world}; each rank's one launch per step TMA-loads the {halo_rows(p)} halo rows "
                   "above/below from its neighbours' HBM (CUDA IPC peer mapping, NVLink), after their per-step "
                   "'input ready' flag; no exchange step")
        else:
            par = f"row strips x{world}, {halo_rows(p)}-row {_backend_name()} halo exchange"
    else:
        par = "single GPU" + (", one launch per step replayed as a CUDA graph" if graph else "")
    l2 = (f"inputs larger than L2 ({in_bytes / 1e6:.0f} MB in + {in_bytes / 1e6:.0f} MB out per step > 126 MB L2); "
          "no flush" if 2 * in_bytes > 126e6 else
          f"scene ({2 * in_bytes / 1e6:.1f} MB in + out) is L2-resident across steps: no flush, "
          "a latency/launch-bound config")
    return {
        "workload": f"{cfg['desc']}; dual LoG (sigma 0.5, 20; 5x5) + {zc} + 5x5 std gate "
                    f"({'on the ZC image' if p.std_source == 0 else 'on the intensity image'}, T={p.std_threshold[0]:g})"
                    f" + OR + {hm}, extract",
        "name": name, "width": W, "height": H, "bit_depth": cfg["bit_depth"], "bands": B,
        "parallelism": par, "l2": l2,
        **({"log_unit": log_unit} if log_unit else {}),
        "params": {"sigma": list(p.sigma), "log_size": list(p.log_size), "zc_threshold": list(p.zc_threshold),
                   "std_source": "zc" if p.std_source == 0 else "intensity", "std_window": p.std_window,
                   "std_threshold": list(p.std_threshold),
                   "hybrid_median": bool(p.hybrid_median), "median_window": p.median_window,
                   "median_window2": p.median_window2, "adaptive": p.adaptive, "out_mode": "extract"},
    }


def _profile_json(name):
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy bandwidth)"
    except Exception:
        return FALLBACK_HBM_GBS, "fallback (B200_PROFILING.md)"


class NvmlSampler:
    """SM clocks and clock-event (throttle) reasons polled through NVML every ~1 ms
    by a background thread DURING the timed region (an in-process query: no
    nvidia-smi start-up latency, so even a 16 ms region gets several samples)."""

    def __init__(self, gpu_index: int):
        import pynvml
        self.nv = pynvml
        pynvml.nvmlInit()
        self.h = pynvml.nvmlDeviceGetHandleByIndex(gpu_index)
        self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        self.rows = []
        self._run = False

    def _poll(self):
        nv = self.nv
        while self._run:
            self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                              nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
            time.sleep(0.001)

    def start(self):
        self._run = True
        self._t = threading.Thread(target=self._poll, daemon=True)
        self._t.start()
        while not self.rows:  # the first sample is in before the timed region starts
            time.sleep(0.0005)
        self.rows.clear()

    def stop(self):
        self._run = False
        self._t.join(1)
        nv = self.nv
        if not self.rows:  # a region shorter than the poll period (c1: ~1 ms): one sample at its end
            self.rows.append((nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM),
                              nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)))
        bits = {"hw_slowdown": nv.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": nv.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": nv.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": nv.nvmlClocksEventReasonSwPowerCap}
        reasons = sorted({n for _, r in self.rows for n, b in bits.items() if r & b})
        sm = [float(c) for c, _ in self.rows]
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": float(self.max_mhz),
                "reasons": reasons, "samples": len(sm), "source": "NVML, polled every 1 ms in the timed region"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region (the
    fallback when NVML is not importable)."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._proc = None

    def start(self):
        try:
            self._proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.gpu}", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except Exception:
            self._proc = None

    def _read(self):
        for line in self._proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def stop(self):
        if self._proc is None:
            return None
        time.sleep(0.25)
        self._proc.terminate()
        try:
            self._proc.wait(2)
        except Exception:
            self._proc.kill()
        self._t.join(1)
        sm = [float(r[1]) for r in self.rows if len(r) >= 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) >= 8 and r[2].replace(".", "").isdigit()]
        reasons = set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            if len(r) >= 8:
                for n, v in zip(names, r[4:8]):
                    if v.lower() == "active":
                        reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_setup(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    share = args.impl == "lfe" and os.environ.get("LFE_BENCH_SHARE_GPUS")
    if share:
        # test hook only: fold ranks onto the visible GPUs (exercises the N > 1 step on one GPU)
        import torch
        local %= max(1, torch.cuda.device_count())
    if world > 1:
        if args.impl == "lfe" and not share:
            # the communicator's INIT lines (nranks, NVLS / P2P transport) go to the log
            os.environ.setdefault("NCCL_DEBUG", "INFO")
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        import torch.distributed as dist
        if args.impl == "lfe":
            import torch
            torch.cuda.set_device(local)  # before the first NCCL call (P2P needs the device set)
        # NCCL refuses two ranks on one GPU: the test hook runs the same step over gloo
        # (shard.py stages the halo rows through host memory)
        dist.init_process_group("nccl" if args.impl == "lfe" and not share else "gloo")
        dist.barrier()  # a full-group collective first: batch_isend_irecv's first call must not be partial
    return world, rank, local


def host_strip_cuts(H, S):
    """The row cuts lfe_extract_host streams (lfe_host.cu host_strip_cuts): S-row
    strips, with S/4- and S/2-row strips at both ends when more than 4 strips."""
    q, hf = max(1, S // 4), max(1, S // 2)
    if H <= 4 * S or q == hf:
        return list(range(0, H, S)) + [H]
    mid = H - 2 * (q + hf)
    n = -(-mid // S)
    return [0, q, q + hf] + [q + hf + mid * k // n for k in range(1, n)] + [H - q - hf, H - q, H]


def all_reduce_dev(t, op=None):
    """all_reduce of a device tensor; through host memory when the group is gloo
    (the one-GPU test hook)."""
    import torch.distributed as dist
    op = dist.ReduceOp.SUM if op is None else op
    if t.is_cuda and dist.get_backend() == "gloo":
        h = t.cpu()
        dist.all_reduce(h, op=op)
        t.copy_(h)
    else:
        dist.all_reduce(t, op=op)
    return t


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            return next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        return "?"


# ------------------------------------------------------------- scenes ----
def c5_check_bands(H=48000, tile=12000, strip=2048):
    """Row bands of the c5 mosaic the oracle checks: the first
    and last rows, every tile seam, and a band across a host-strip boundary in
    every tile row (tests/test_gpu_parity.py uses the same bands)."""
    bands = [(0, 16), (H - 16, H)]
    bands += [(s - 10, s + 10) for s in range(tile, H, tile)]
    bands += [(t * tile + 5 * strip - 8, t * tile + 5 * strip + 8) for t in range(H // tile)]
    return bands


class Scene:
    """Host rows of a single-image config: c1-c3 generated whole; c5 (4.6 GB) only
    the rows one rank holds, generated tile by tile into pinned host memory."""

    def __init__(self, name, cfg):
        self.name, self.cfg = name, cfg
        self._img, self._r0 = None, 0

    def hold(self, a, b, pinned=False):
        """Generate (or keep) rows [a, b); later rows() calls must fall inside them."""
        import numpy as np
        import torch
        from paper_1304_3992_b200 import scenes
        if self.name == "c1":
            img = scenes.scene_c1()
        elif self.name == "c2":
            img = scenes.scene_c2()
        elif self.name == "c3":
            img = scenes.scene_c3(size=self.cfg["W"])
        else:
            dt = torch.uint16
            self._pinned = torch.empty((b - a, self.cfg["W"]), dtype=dt, pin_memory=pinned)
            scenes.scene_c5_rows(a, b, out=self._pinned.numpy())
            self._img, self._r0 = self._pinned.numpy(), a
            return
        self._img, self._r0 = np.ascontiguousarray(img), 0

    def rows(self, a, b):
        a0 = a - self._r0
        if a0 < 0 or b - self._r0 > self._img.shape[0]:
            raise IndexError(f"rows [{a}, {b}) not held")
        return self._img[a0:b - self._r0]


# ------------------------------------------------------------- oracle legs ----
def oracle_rows(scene, p, a, b):
    """The oracle on owned rows [a, b) of a single-image scene (plus real halo
    rows, clamped only at the true image edge): returns the (b - a) output rows."""
    import numpy as np
    import oracle
    H = scene.cfg["H"]
    h = halo_rows(p)
    lo, hi = max(0, a - h), min(H, b + h)
    ref = oracle.run(np.ascontiguousarray(scene.rows(lo, hi)), oracle_params(p))
    return ref[a - lo:b - lo]


def parity_bands(name, a, b):
    """The owned row bands [a, b) of a rank that the oracle checks."""
    if name != "c5":
        return [(a, b)]
    out = []
    for x, y in c5_check_bands():
        x, y = max(x, a), min(y, b)
        if x < y:
            out.append((x, y))
    return out


def timed_oracle(fn, min_s=0.0):
    """Run fn() (at least once, repeating until min_s seconds); (result, seconds per run)."""
    t0 = time.perf_counter()
    n, res = 0, None
    while True:
        res = fn()
        n += 1
        dt = time.perf_counter() - t0
        if dt >= min_s:
            return res, dt / n


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle, as it stands, on the same config: each
    step a 512-row, full-width sample of the scene (all 512 rows for c1; for c4
    one band per step, cycling)."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    from paper_1304_3992_b200 import scenes
    cfg = geometry(args)
    p = workload_params(cfg, args.median2, args.adaptive, args.std)
    H, W, h = cfg["H"], cfg["W"], halo_rows(p)
    rows = min(512, H)
    if args.config == "c4":
        sc = scenes.scene_c4(size=W)
        get = lambda i, lo, hi: sc[i % 4, lo:hi]  # noqa: E731
    elif args.config == "c5":
        tile_row = scenes.scene_c5_rows(0, 12000)  # the samples come from the mosaic's first tile row
        H = 12000
        get = lambda i, lo, hi: tile_row[lo:hi]  # noqa: E731
    else:
        sc = Scene(args.config, cfg)
        sc.hold(0, H)
        get = lambda i, lo, hi: sc.rows(lo, hi)  # noqa: E731
    op = oracle_params(p)
    times = []
    for i in range(args.warmup + args.steps):
        a = (H // 2 - rows // 2 + 977 * i) % (H - rows) if H > rows else 0
        band = np.ascontiguousarray(get(i, max(0, a - h), min(H, a + rows + h)))
        t0 = time.perf_counter()
        oracle.run(band, op)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = rows * W * len(times) / tot / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(times), 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": config_dict(args.config, cfg, world, p),
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": oracle.get_threads(), "kind": "oracle",
                             "sample": f"each step: {rows} x {W} rows of {args.config} (+{h} halo rows), "
                                       "plain C oracle -O2 OpenMP over rows", "cpu_model": cpu_model()},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


# ------------------------------------------------------------------ main ----
def main():
    args = parse()
    world, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, world, rank)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return

    import numpy as np
    import torch

    import paper_1304_3992_b200.shard as shard_mod
    from paper_1304_3992_b200 import lfe, scenes

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = geometry(args)
    name = args.config
    p = workload_params(cfg, args.median2, args.adaptive, args.std)
    H, W, NB = cfg["H"], cfg["W"], cfg["bands"]
    tdt = torch.uint8 if elem(cfg) == 1 else torch.uint16
    esz = elem(cfg)
    ctx = lfe.Context(p)
    ctx.set_option(lfe.LFE_OPT_KERNEL, {"auto": 0, "staged": 1, "fused": 2}[args.kernel])
    ctx.set_option(lfe.LFE_OPT_LOG_UNIT, {"auto": lfe.LFE_LOG_AUTO, "cuda": lfe.LFE_LOG_CUDA_CORES,
                                          "tensor": lfe.LFE_LOG_TENSOR_CORES}[args.log_unit])
    if args.tile:
        tw, th = (int(v) for v in args.tile.split("x"))
        ctx.set_option(lfe.LFE_OPT_TILE_W, tw)
        ctx.set_option(lfe.LFE_OPT_TILE_H, th)
    halo = ctx.halo
    assert halo == halo_rows(p)
    kernel_events = []
    use_graph = name in ("c1", "c2") and world == 1 and not args.no_graph and not p.adaptive

    def cur_stream():
        return torch.cuda.current_stream(dev)

    def rec(record, fn, px):
        if record:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(cur_stream())
        fn()
        if record:
            e1.record(cur_stream())
            kernel_events.append((e0, e1, px))

    # ---------------- device buffers and the step ----------------
    import torch.distributed as dist  # noqa: F401 (N > 1 only)
    halo_mode = None
    if NB > 1:  # c4: bands
        bs = shard_mod.BandShard(NB, H, W, rank, world, halo)
        bs.alloc(tdt, dev)
        scene4 = scenes.scene_c4(size=W)
        bs.load_owned(scene4)
        whole_out = torch.empty_like(bs.whole_buf) if bs.whole else None
        part_outs = [torch.empty((e - a, W), dtype=tdt, device=dev) for _, a, e, _, _ in bs.parts]
        calls = bs.part_calls()
        owned_px = bs.owned_pixels()

        def step(record=False):
            works = bs.exchange() if world > 1 and bs.parts else []
            sp = cur_stream().cuda_stream
            if bs.whole:
                wb, wo = bs.whole_buf, whole_out
                rec(record, lambda: lfe.lfe_extract_bands(
                    ctx.handle, wb.data_ptr(), wb.stride(1) * esz, wb.stride(0) * esz, W, H, wb.shape[0],
                    wo.data_ptr(), wo.stride(1) * esz, wo.stride(0) * esz, sp), wb.shape[0] * H * W)
            waited = False
            for k, s, n, ha, hb, flags, need in calls:
                if need and not waited:
                    for w in works:
                        w.wait()
                    waited = True
                buf, o = bs.part_bufs[k], part_outs[k]
                row0 = (0 if bs.parts[k][3] is None else halo) + s  # buffer row of owned row s
                rec(record, lambda buf=buf, o=o, row0=row0, n=n, ha=ha, hb=hb, flags=flags, s=s: lfe.lfe_extract_rows(
                    ctx.handle, buf.data_ptr() + row0 * buf.stride(0) * esz, buf.stride(0) * esz, W, n, ha, hb,
                    flags, o.data_ptr() + s * o.stride(0) * esz, o.stride(0) * esz, sp), n * W)
            if not waited:
                for w in works:
                    w.wait()
    elif world > 1 and args.halo != "nccl" and not p.adaptive:
        # peer halos: every rank holds only its owned rows; one launch per step reads the
        # neighbours' boundary rows in place (their HBM over NVLink), after their "input
        # ready" flag for this step
        scene = Scene(name, cfg)
        shard = shard_mod.PeerStripShard(H, W, rank, world, halo)
        buf = shard.alloc(tdt, dev)
        scene.hold(shard.a - shard.ha, shard.b + shard.hb, pinned=not args.no_e2e)
        buf.copy_(torch.from_numpy(scene.rows(shard.a, shard.b)))
        out = torch.empty((shard.rows, W), dtype=tdt, device=dev)
        torch.cuda.synchronize(dev)
        shard.connect()
        da, pa, db, pb, fa, fb = shard.call_args()
        share = bool(os.environ.get("LFE_BENCH_SHARE_GPUS"))
        if share:
            # ranks sharing one GPU time-slice between processes: signal once, up front,
            # so that no kernel ever spins on a neighbour that cannot run
            lfe.lfe_signal(shard.flag.data_ptr(), 1 << 62, cur_stream().cuda_stream)
            torch.cuda.synchronize(dev)
        dist.barrier()  # every rank's rows are in place before any neighbour reads them
        owned_px = shard.rows * W
        counter = [0]
        bpitch, opitch = buf.stride(0) * esz, out.stride(0) * esz
        halo_mode = "peer"

        def step(record=False):
            counter[0] += 1
            v = 1 if share else counter[0]
            sp = cur_stream().cuda_stream
            if not share:  # this step's input is in place: neighbours may read it
                lfe.lfe_signal(shard.flag.data_ptr(), v, sp)
            rec(record, lambda: lfe.lfe_extract_rows_peer(
                ctx.handle, buf.data_ptr(), bpitch, W, shard.rows, da, pa, db, pb, shard.edge_flags(), fa, fb, v,
                out.data_ptr(), opitch, sp), owned_px)
    else:
        halo_mode = "nccl"
        scene = Scene(name, cfg)
        shard = shard_mod.StripShard(H, W, rank, world, halo)
        buf = shard.alloc(tdt, dev)
        # this rank's rows plus the halo rows its neighbours send (c5: only the tiles they cross)
        scene.hold(shard.a - shard.ha, shard.b + shard.hb, pinned=not args.no_e2e)
        buf.copy_(torch.from_numpy(scene.rows(shard.a - shard.ha, shard.b + shard.hb)))
        out = torch.empty((shard.rows, W), dtype=tdt, device=dev)
        bpitch, opitch = buf.stride(0) * esz, out.stride(0) * esz
        bands = shard.bands()
        stats = torch.zeros(9, dtype=torch.int64, device=dev) if p.adaptive else None
        owned_px = shard.rows * W

        def launch(band, record):
            s, n, ha, hb, flags, _ = band
            sp = cur_stream().cuda_stream
            rec(record, lambda: lfe.lfe_extract_rows(ctx.handle, buf.data_ptr() + (shard.ha + s) * bpitch, bpitch, W,
                                                     n, ha, hb, flags, out.data_ptr() + s * opitch, opitch, sp),
                n * W)

        def step(record=False):
            works = shard.exchange() if world > 1 else []
            if p.adaptive:  # NEXT-2: whole-scene statistics first (needs the halo rows), one sync
                for w in works:
                    w.wait()
                works = []
                stats.zero_()
                lfe.lfe_stats_rows(ctx.handle, buf.data_ptr() + shard.ha * bpitch, bpitch, W, shard.rows, shard.ha,
                                   shard.hb, shard.edge_flags(), stats.data_ptr(), cur_stream().cuda_stream)
                shard.allreduce_stats(stats)
                ctx.set_stats_device(stats)  # resolved on the device: no host round trip
            for b in bands:
                if not b[5]:
                    launch(b, record)
            for w in works:
                w.wait()
            for b in bands:
                if b[5]:
                    launch(b, record)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    ctx.check()

    graph = None
    launches_per_step = None
    if use_graph:  # c1 / c2: the step (one launch) captured once, replayed per step
        n0 = ctx.launches
        graph = torch.cuda.CUDAGraph()
        gs = torch.cuda.Stream(dev)
        gs.wait_stream(cur_stream())
        with torch.cuda.stream(gs):
            with torch.cuda.graph(graph, stream=gs):
                step()
        cur_stream().wait_stream(gs)
        launches_per_step = ctx.launches - n0
        for _ in range(3):
            graph.replay()
        torch.cuda.synchronize(dev)
        ctx.check()

    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    try:
        clocks = NvmlSampler(local)
    except Exception:
        clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.launches
    stream = cur_stream()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    t0.record(stream)
    for _ in range(args.steps):
        if graph is not None:
            rec(True, graph.replay, owned_px)
        else:
            step(record=True)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    launches = (ctx.launches - launches0) if graph is None else launches_per_step * args.steps
    ms = t0.elapsed_time(t1)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device=dev)
        all_reduce_dev(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        dist.barrier()
    ctx.check()

    # dominant kernel: the launch with the most pixels (the interior band / all whole
    # bands); average duration over the timed steps
    main_px = max(n for _, _, n in kernel_events)
    kms = [a.elapsed_time(b) for a, b, n in kernel_events if n == main_px]
    k_ms = sum(kms) / len(kms)
    bytes_launch = main_px * (esz + esz)  # input read once + output written once (EXTRACT: same dtype)
    achieved = bytes_launch / (k_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    # ---------------- parity of the last timed step (before anything else reuses `out`) ----------------
    parity = None
    cpu = None
    if not args.no_parity:
        import oracle
        cores = oracle.get_threads()
        if world > 1:  # ranks share the host's cores
            oracle.set_threads(max(1, (os.cpu_count() or 1) // world))
        diff, cmp_px = 0, 0
        t_or = time.perf_counter()
        if NB > 1:
            op = oracle_params(p)
            if bs.whole:
                got = whole_out.cpu().numpy()
                for i, b in enumerate(bs.whole):
                    want = oracle.run(scene4[b], op)
                    diff += int((got[i] != want).sum())
                    cmp_px += want.size
            for (b, a, e, _, _), o in zip(bs.parts, part_outs):
                lo, hi = max(0, a - halo), min(H, e + halo)
                want = oracle.run(np.ascontiguousarray(scene4[b, lo:hi]), op)[a - lo:e - lo]
                diff += int((o.cpu().numpy() != want).sum())
                cmp_px += want.size
        else:
            for a, b in ([] if p.adaptive else parity_bands(name, shard.a, shard.b)):
                want = oracle_rows(scene, p, a, b)
                got = out[a - shard.a:b - shard.a].cpu().numpy()
                diff += int((got != want).sum())
                cmp_px += want.size
        t_or = time.perf_counter() - t_or
        oracle.set_threads(cores)
        pt = torch.tensor([diff, cmp_px], dtype=torch.int64, device=dev)
        if world > 1:
            all_reduce_dev(pt)
        diff, cmp_px = (int(v) for v in pt.tolist())
        if cmp_px:
            parity = {"pixels": cmp_px, "differing": diff, "bit_exact": diff == 0,
                      "vs": "CPU oracle (oracle/lfe_oracle.c), output of the last timed step",
                      "scope": ("whole scene" if name != "c5" else
                                f"{len(c5_check_bands())} full-width row bands: first/last rows, every tile seam, "
                                "a host-strip boundary in every tile row")}
        if rank == 0 and world == 1 and cmp_px and not args.no_cpu_baseline:
            # the same oracle run, timed: the CPU baseline (the oracle as it stands)
            cpu = {"value": round(cmp_px / t_or / 1e6, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
                   "sample": f"{parity['scope']} of {name} ({cmp_px} output px, + halo rows), one run, "
                             f"{t_or:.2f} s, plain C oracle -O2 OpenMP over rows (the parity check's own run)",
                   "cpu_model": cpu_model(), "host_cpus": os.cpu_count()}
        if p.adaptive:
            parity = {"skipped": "adaptive: GPU-test covered (test_adaptive_c3_full_size)"}

    # ---------------- end to end through the public API with host buffers (pinned) ----------------
    e2e = None
    if not args.no_e2e:
        K = max(1, min(args.steps, 10 if name != "c5" else 2))
        strip_rows = 1024 if name != "c5" else 2048
        ctx.set_option(lfe.LFE_OPT_HOST_STRIP_ROWS, strip_rows)
        if NB > 1:
            # every owned band (or cut piece plus its neighbours' halo rows) from host memory
            pieces = [(b, 0, H, 0, H) for b in bs.whole] + [
                (b, a, e, max(0, a - halo), min(H, e + halo)) for b, a, e, _, _ in bs.parts]
        else:
            pieces = [(0, shard.a, shard.b, shard.a - shard.ha, shard.b + shard.hb)]
        h_in, h_out = [], []
        for b, a, e, ea, eb in pieces:
            hi = torch.empty((eb - ea, W), dtype=tdt, pin_memory=True)
            hi.numpy()[...] = scene4[b, ea:eb] if NB > 1 else scene.rows(ea, eb)
            h_in.append(hi)
            h_out.append(torch.empty((eb - ea, W), dtype=tdt, pin_memory=True))

        def e2e_step():
            for hi, ho in zip(h_in, h_out):
                ctx.extract_host_ptr(hi.data_ptr(), W * esz, W, hi.shape[0], ho.data_ptr(), W * esz)

        e2e_step()  # warm-up
        if world > 1:
            dist.barrier()
        tw0 = time.perf_counter()
        for _ in range(K):
            e2e_step()
        e2e_s = time.perf_counter() - tw0
        if world > 1:
            tt = torch.tensor([e2e_s], device=dev)
            all_reduce_dev(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        h2d_rows = 0
        for hi in h_in:
            rows_e = hi.shape[0]
            cuts = host_strip_cuts(rows_e, strip_rows)
            h2d_rows += sum(min(rows_e, b + halo) - max(0, a - halo) for a, b in zip(cuts, cuts[1:]))
        h2d_tot = torch.tensor([h2d_rows * W * esz, sum(x.shape[0] for x in h_out) * W * esz], dtype=torch.int64,
                               device=dev)
        if world > 1:
            all_reduce_dev(h2d_tot)
        h2d_b, d2h_b = (int(v) for v in h2d_tot.tolist())
        e2e = {"value": round(NB * H * W * K / e2e_s / 1e6, 3), "unit": UNIT,
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
               "how": "lfe_extract_host on pinned host buffers: strip-pipelined H2D -> kernel -> D2H on 3 streams, "
                      f"{strip_rows}-row strips ({strip_rows // 4} and {strip_rows // 2} rows at both ends), wall clock "
                      f"of {K} synchronous steps (max over ranks); each rank streams its rows plus its neighbours' "
                      "halo rows" + ("; one call per band" if NB > 1 else "")}
        del h_in, h_out

    verify = None
    if args.verify:  # the last timed step's owned rows == a whole-scene extraction on this GPU
        whole = ctx.extract(torch.from_numpy(np.ascontiguousarray(scene.rows(0, H))).to(dev))
        ctx.check()
        bad = torch.tensor([int((out != whole[shard.a:shard.b]).sum().item())], dtype=torch.int64, device=dev)
        if world > 1:
            all_reduce_dev(bad)
        verify = {"bit_exact_vs_whole_scene": int(bad.item()) == 0, "differing_pixels": int(bad.item())}
        del whole

    if rank == 0:
        value = NB * H * W * args.steps / (ms * 1e-3) / 1e6
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": config_dict(name, cfg, world, p, graph=graph is not None, halo_mode=halo_mode,
                                  log_unit=log_unit_of(ctx, p, args.log_unit,
                                                       NB * ((W + 1343) // 1344) * (H // world))),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": None,
                         "kernel": "lfe fused stencil kernel (dominant launch: the interior band / all whole bands)"
                                   + ("; graph replay of the one-launch step" if graph is not None else ""),
                         "kernel_ms": round(k_ms, 4), "algorithmic_bytes_per_launch": bytes_launch,
                         "bytes_per_px": 2 * esz, "peak_source": peak_src},
            "parity": parity,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "cpu_baseline": cpu,
            "clocks": clk,
            "paper_context": {"note": "other hardware (Tesla C2075 vs Xeon E5620), context only",
                              "paper_gpu_kernel_mpx_s": 43.0, "paper_gpu_kernel_workload": "Cartosat-1 4000x4000, "
                              "urban (Table 6, PAPER.md:226)", "paper_speedup": "20.7x GPU vs 2-thread CPU "
                              "(AWiFS, Table 7, PAPER.md:236)",
                              "this_gpu_vs_oracle": round(value / cpu["value"], 1) if cpu else None,
                              # the paper's convention: % speed-up = (T_cpu / T_gpu - 1) x 100
                              "this_gpu_vs_oracle_pct_speedup": round((value / cpu["value"] - 1) * 100) if cpu else None},
        }
        if verify is not None:
            line["verify"] = verify
        src = fused_source_hash()
        headline = name == "c3" and cfg["W"] == 12000 and not p.adaptive and not p.median_window2 \
            and args.kernel != "staged" and args.std == "zc"
        iss = _profile_json("issue.json")
        if iss and headline:
            # the binding resource: instruction issue, 4 warp-instructions
            # per clock per SM = 148 * 4 * 32 lane-ops per clock at the SM clock under load
            mhz = (clk or {}).get("sm_mhz") or 1965.0
            ach = iss["inst_per_launch"] * 32 / (k_ms * 1e-3) / 1e12
            pk = 148 * 4 * 32 * mhz * 1e6 / 1e12
            line["issue"] = {"bound": "alu", "achieved": round(ach, 2), "peak": round(pk, 2),
                             "unit": "Tlane-op/s issued", "frac": round(ach / pk, 4),
                             "inst_per_launch": iss["inst_per_launch"], "sm_mhz": mhz,
                             "source": iss.get("source"), "source_sha": iss.get("source_sha"),
                             "matches_kernel_source": iss.get("source_sha") == src}
        tr = _profile_json("traffic.json")
        if tr and headline:
            ok = tr.get("source_sha") == src
            line["roofline"]["traffic"] = tr.get("bytes_per_launch") if ok else None
            line["roofline"]["traffic_source"] = tr.get("source")
            line["roofline"]["traffic_matches_kernel_source"] = ok
            if not ok:
                line["roofline"]["traffic_stale"] = tr.get("bytes_per_launch")
        line["kernel_source_sha"] = src
        print(json.dumps(line), flush=True)
    if halo_mode == "peer":
        torch.cuda.synchronize(dev)
        dist.barrier()  # no neighbour reads this rank's rows any more
        shard.close()
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
