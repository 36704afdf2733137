#!/usr/bin/env python
"""Benchmark of the dual-LoG feature-extraction hot path (arXiv 1304.3992) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl lfe|reference]

A step = one pass of the whole hot path (LoG x2 -> zero crossing -> std gate ->
OR merge -> hybrid median) over the c3 scene: 12000 x 12000 uint16 (10-bit),
Cartosat-1-like synthetic PAN, resident in HBM.  At N > 1 (torchrun, one
process per GPU) the scene is split into N row strips with an NCCL halo
exchange of 7 boundary rows per neighbour (strong scaling: the scene is fixed).
--median2 3 adds the water pipeline's second median level (8-row halo).
Rank 0 prints one JSON line.  See DESIGN.md "Measurement".
"""
from __future__ import annotations

import argparse
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


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", choices=["lfe", "reference"], default="lfe")
    ap.add_argument("--kernel", choices=["auto", "staged", "fused"], default="auto")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--verify", action="store_true",
                    help="after timing, check every rank's owned output rows against a whole-scene "
                         "extraction on its own GPU (bit-exact); adds \"verify\" to the line")
    ap.add_argument("--size", type=int, default=12000, help="scene side (default: c3's 12000)")
    ap.add_argument("--tile", type=str, default="", help="TWxTH override (tuning only)")
    ap.add_argument("--median2", type=int, default=0, choices=[0, 3, 5, 7],
                    help="second hybrid-median level (the water pipeline, PAPER.md:102); 0 = the c3 metric config")
    ap.add_argument("--adaptive", type=float, default=0.0,
                    help="k > 0: adaptive ZC gap t = ceil(k * sigma(r)) (SPEC.md:233, NEXT-2), with its "
                         "statistics pre-pass and all-reduce inside every step; 0 = the c3 metric config")
    return ap.parse_args()


def workload_params(median2=0, adaptive=0.0):
    from paper_1304_3992_b200 import lfe
    # SURVEY.md 8(c) defaults for benchmark scenes: ZC gap 0.02 (normalised),
    # std source = ZC image, 5x5 window, T = 0.3, hybrid median on, extract.
    zc = (adaptive, adaptive) if adaptive > 0 else (0.02, 0.02)
    return lfe.Params(bit_depth=10, sigma=(0.5, 20.0), log_size=(5, 5), zc_threshold=zc,
                      std_source=lfe.LFE_STD_ZC, std_window=5, std_threshold=(0.3, 0.3),
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


def _backend_name():
    try:
        import torch.distributed as dist
        b = dist.get_backend() if dist.is_initialized() else "nccl"
    except Exception:
        b = "nccl"
    return "NCCL" if b == "nccl" else f"{b} (host-staged; ranks sharing a GPU: test hook, not a measurement)"


def config_dict(size, world, p):
    hm = "5x5 hybrid median" + (f" + {p.median_window2}x{p.median_window2} second level" if p.median_window2 else "")
    zc = (f"ZC (adaptive gap {p.zc_threshold[0]} x global std of r, statistics pre-pass)" if p.adaptive
          else "ZC (gap 0.02)")
    return {
        "workload": f"c3: {size}x{size} uint16 (10-bit) synthetic Cartosat-1-like PAN scene, "
                    f"dual LoG (sigma 0.5, 20; 5x5) + {zc} + 5x5 std gate (T=0.3) + OR + {hm}, extract",
        "width": size, "height": size, "bit_depth": 10, "bands": 1,
        "parallelism": (f"row strips x{world}, {halo_rows(p)}-row {_backend_name()} halo exchange" if world > 1
                        else "single GPU"),
        "l2": "inputs larger than L2 (288 MB in + 288 MB out per step > 126 MB L2); no flush",
        "params": {"sigma": list(p.sigma), "log_size": list(p.log_size), "zc_threshold": list(p.zc_threshold),
                   "std_source": "zc", "std_window": p.std_window, "std_threshold": list(p.std_threshold),
                   "hybrid_median": bool(p.hybrid_median), "median_window": p.median_window,
                   "median_window2": p.median_window2, "adaptive": p.adaptive, "out_mode": "extract"},
    }


def ncu_issue():
    """Executed warp-instructions per launch of the dominant kernel (committed
    ncu summary, profiles/issue.json), or None."""
    try:
        with open(os.path.join(ROOT, "profiles", "issue.json")) as f:
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


def ncu_traffic():
    """DRAM bytes per launch of the dominant kernel from the committed ncu
    --set full summary (profiles/), or None."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as f:
            return json.load(f)
    except Exception:
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.rows = []
        self._stop = threading.Event()
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
    if args.impl == "lfe" and os.environ.get("LFE_BENCH_SHARE_GPUS"):
        # test hook only: fold ranks onto the visible GPUs (exercises the N > 1 step on one GPU)
        import torch
        local %= max(1, torch.cuda.device_count())
    if world > 1:
        import torch.distributed as dist
        if args.impl == "lfe":
            import torch
            torch.cuda.set_device(local)  # before the first NCCL call (P2P needs the device set)
        share = args.impl == "lfe" and os.environ.get("LFE_BENCH_SHARE_GPUS")
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


def cpu_baseline(img, p, rows=None):
    """The oracle as it stands, on the host cores, on a bounded sample of the
    same workload: `rows` full-width rows (+ halo rows each side); default the
    whole scene (about 6 s on 16 cores)."""
    import oracle
    H = img.shape[0]
    h = halo_rows(p)
    rows = H if rows is None else min(rows, H)
    a = H // 2 - rows // 2
    lo, hi = max(0, a - h), min(H, a + rows + h)
    band = img[lo:hi].copy()
    op = oracle_params(p)
    t0 = time.perf_counter()
    oracle.run(band, op)
    dt = time.perf_counter() - t0
    px = rows * img.shape[1]  # output rows counted (halo rows are overhead)
    # single-thread leg on a small bounded sample
    cores = oracle.get_threads()
    r1 = min(192, H)
    a1 = H // 2 - r1 // 2
    b1 = img[max(0, a1 - h):min(H, a1 + r1 + h)].copy()
    oracle.set_threads(1)
    t1 = time.perf_counter()
    oracle.run(b1, op)
    d1 = time.perf_counter() - t1
    oracle.set_threads(cores)
    model = "?"
    try:
        with open("/proc/cpuinfo") as f:
            model = next(l.split(":", 1)[1].strip() for l in f if l.startswith("model name"))
    except Exception:
        pass
    return {"value": round(px / dt / 1e6, 3), "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{rows} x {img.shape[1]} rows of the c3 scene (+{h} halo rows each side), one run, "
                      f"{dt:.2f} s, plain C oracle -O2 OpenMP over rows",
            "single_thread": {"value": round(r1 * img.shape[1] / d1 / 1e6, 3), "unit": UNIT,
                              "sample": f"{r1} x {img.shape[1]} rows, 1 thread, {d1:.2f} s"},
            "cpu_model": model, "host_cpus": os.cpu_count()}


def run_reference(args, world, rank):
    """--impl reference: the CPU oracle, as it stands, on the same config."""
    if rank != 0:
        return
    import numpy as np

    import oracle
    from paper_1304_3992_b200 import scenes
    p = workload_params(args.median2, args.adaptive)
    img = scenes.scene_c3(size=args.size)
    rows = 512
    H, W = img.shape
    h = halo_rows(p)
    op = oracle_params(p)
    times = []
    for i in range(args.warmup + args.steps):
        a = (H // 2 - rows // 2 + 977 * i) % (H - rows)
        band = np.ascontiguousarray(img[max(0, a - h):min(H, a + rows + h)])
        t0 = time.perf_counter()
        oracle.run(band, op)
        if i >= args.warmup:
            times.append(time.perf_counter() - t0)
    tot = sum(times)
    value = rows * W * len(times) / tot / 1e6
    line = {"impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(1e3 * tot / len(times), 3),
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "int64",
            "data": "synthetic", "config": config_dict(args.size, world, p),
            "cpu_baseline": {"value": round(value, 3), "unit": UNIT, "cores": oracle.get_threads(), "kind": "oracle",
                             "sample": f"each step: {rows} x {W} rows of c3 (+{h} halo rows), plain C oracle -O2 OpenMP"},
            "e2e": {"value": round(value, 3), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "gpu_launches": 0}
    print(json.dumps(line), flush=True)


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

    from paper_1304_3992_b200 import lfe, scenes
    from paper_1304_3992_b200.shard import StripShard

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    p = workload_params(args.median2, args.adaptive)
    size = args.size
    img = scenes.scene_c3(size=size)                      # host, numpy uint16
    H, W = img.shape
    ctx = lfe.Context(p)
    ctx.set_option(lfe.LFE_OPT_KERNEL, {"auto": 0, "staged": 1, "fused": 2}[args.kernel])
    if args.tile:
        tw, th = (int(v) for v in args.tile.split("x"))
        ctx.set_option(lfe.LFE_OPT_TILE_W, tw)
        ctx.set_option(lfe.LFE_OPT_TILE_H, th)
    halo = ctx.halo
    assert halo == halo_rows(p)
    shard = StripShard(H, W, rank, world, halo)
    buf = shard.alloc(torch.uint16, dev)
    shard.load_owned(img)
    out = torch.empty((shard.rows, W), dtype=torch.uint16, device=dev)
    stream = torch.cuda.current_stream(dev)
    sptr = stream.cuda_stream
    bpitch, opitch = buf.stride(0) * 2, out.stride(0) * 2
    kernel_events = []

    def launch(band, record):
        s, n, ha, hb, flags, _ = band
        if record:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
        lfe.lfe_extract_rows(ctx.handle, buf.data_ptr() + (shard.ha + s) * bpitch, bpitch, W, n, ha, hb, flags,
                             out.data_ptr() + s * opitch, opitch, sptr)
        if record:
            e1.record(stream)
            kernel_events.append((e0, e1, n))

    bands = shard.bands()
    stats = torch.zeros(9, dtype=torch.int64, device=dev) if p.adaptive else None

    def step(record=False):
        works = shard.exchange() if world > 1 else []
        if p.adaptive:  # NEXT-2: whole-scene statistics first (needs the halo rows), one sync
            for w in works:
                w.wait()
            works = []
            stats.zero_()
            lfe.lfe_stats_rows(ctx.handle, buf.data_ptr() + shard.ha * bpitch, bpitch, W, shard.rows, shard.ha,
                               shard.hb, shard.edge_flags(), stats.data_ptr(), sptr)
            shard.allreduce_stats(stats)
            ctx.set_stats(stats.cpu().tolist())
        for b in bands:
            if b[5]:
                continue
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
    if world > 1:
        import torch.distributed as dist
        dist.barrier()
    clocks = ClockSampler(local)
    clocks.start()
    launches0 = ctx.launches
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    t0.record(stream)
    for _ in range(args.steps):
        step(record=True)
    t1.record(stream)
    torch.cuda.synchronize(dev)
    clk = clocks.stop()
    launches = ctx.launches - launches0
    ms = t0.elapsed_time(t1)
    if world > 1:
        import torch.distributed as dist
        tt = torch.tensor([ms], device=dev)
        all_reduce_dev(tt, op=dist.ReduceOp.MAX)
        ms = float(tt.item())
        dist.barrier()
    ctx.check()

    # dominant kernel: the full-strip launch (interior band); average duration
    main_n = max(n for _, _, n in kernel_events)
    kms = [a.elapsed_time(b) for a, b, n in kernel_events if n == main_n]
    k_ms = sum(kms) / len(kms)
    px_launch = main_n * W
    bytes_launch = px_launch * (2 + 2)  # input read once + output written once (u16 -> u16)
    achieved = bytes_launch / (k_ms * 1e-3) / 1e9
    peak, peak_src = measured_peak()

    # end-to-end through the public API with host buffers (pinned): each rank streams its
    # strip plus the halo rows of its neighbours (so its owned rows are exact) and keeps
    # the owned output rows
    e2e = None
    if not args.no_e2e:
        ea, eb = shard.a - shard.ha, shard.b + shard.hb
        erows = eb - ea
        h_in = torch.from_numpy(np.ascontiguousarray(img[ea:eb])).pin_memory()
        h_out = torch.empty((erows, W), dtype=torch.uint16).pin_memory()
        K = max(1, min(args.steps, 10))
        strip_rows = 1024
        ctx.set_option(lfe.LFE_OPT_HOST_STRIP_ROWS, strip_rows)
        ctx.extract_host_ptr(h_in.data_ptr(), W * 2, W, erows, h_out.data_ptr(), W * 2)  # warm-up
        if world > 1:
            dist.barrier()
        tw0 = time.perf_counter()
        for _ in range(K):
            ctx.extract_host_ptr(h_in.data_ptr(), W * 2, W, erows, h_out.data_ptr(), W * 2)
        e2e_s = time.perf_counter() - tw0
        if world > 1:
            tt = torch.tensor([e2e_s], device=dev)
            all_reduce_dev(tt, op=dist.ReduceOp.MAX)
            e2e_s = float(tt.item())
        cuts = host_strip_cuts(erows, strip_rows)
        h2d_rows = sum(min(erows, b + halo) - max(0, a - halo) for a, b in zip(cuts, cuts[1:]))
        h2d_tot = torch.tensor([h2d_rows * W * 2, erows * W * 2], dtype=torch.int64, device=dev)
        if world > 1:
            all_reduce_dev(h2d_tot)
        h2d_b, d2h_b = (int(v) for v in h2d_tot.tolist())
        e2e = {"value": round(H * W * K / e2e_s / 1e6, 3), "unit": UNIT,
               "h2d_bytes_per_step": h2d_b, "d2h_bytes_per_step": d2h_b,
               "how": "lfe_extract_host on pinned host buffers: strip-pipelined H2D -> kernel -> D2H on 3 streams, "
                      f"{strip_rows}-row strips ({strip_rows // 4} and {strip_rows // 2} rows at both ends), wall clock of {K} synchronous calls (max over ranks); each rank "
                      "streams its strip plus its neighbours' halo rows"}

    verify = None
    if args.verify:  # the last timed step's owned rows == a whole-scene extraction on this GPU
        whole = ctx.extract(torch.from_numpy(img).to(dev))
        ctx.check()
        bad = torch.tensor([int((out != whole[shard.a:shard.b]).sum().item())], dtype=torch.int64, device=dev)
        if world > 1:
            all_reduce_dev(bad)
        verify = {"bit_exact_vs_whole_scene": int(bad.item()) == 0, "differing_pixels": int(bad.item())}
        del whole

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(img, p)

    if rank == 0:
        value = H * W * args.steps / (ms * 1e-3) / 1e6
        line = {
            "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "int32", "data": "synthetic",
            "config": config_dict(size, world, p),
            "roofline": {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                         "frac": round(achieved / peak, 4), "traffic": None,
                         "kernel": "lfe fused/staged stencil kernel (dominant; one launch per step at N=1)",
                         "kernel_ms": round(k_ms, 4), "algorithmic_bytes_per_launch": bytes_launch,
                         "bytes_per_px": 4, "peak_source": peak_src},
            "e2e": e2e,
            "gpu_launches": int(launches),
            "cpu_baseline": cpu,
            "clocks": clk,
            "paper_context": {"note": "other hardware (Tesla C2075 vs Xeon E5620), context only",
                              "paper_gpu_kernel_mpx_s": 43.0, "paper_gpu_kernel_workload": "Cartosat-1 4000x4000, "
                              "urban (Table 6, PAPER.md:226)", "paper_speedup": "20.7x GPU vs 2-thread CPU "
                              "(AWiFS, Table 7, PAPER.md:236)",
                              "this_gpu_vs_oracle": round(value / cpu["value"], 1) if cpu else None},
        }
        if verify is not None:
            line["verify"] = verify
        iss = ncu_issue()
        if iss and not p.adaptive and not p.median_window2:
            # the binding resource: instruction issue, 4 warp-instructions
            # per clock per SM = 148 * 4 * 32 lane-ops per clock at the SM clock under load
            mhz = (clk or {}).get("sm_mhz") or 1965.0
            ach = iss["inst_per_launch"] * 32 / (k_ms * 1e-3) / 1e12
            pk = 148 * 4 * 32 * mhz * 1e6 / 1e12
            line["issue"] = {"bound": "alu", "achieved": round(ach, 2), "peak": round(pk, 2),
                             "unit": "Tlane-op/s issued", "frac": round(ach / pk, 4),
                             "inst_per_launch": iss["inst_per_launch"], "sm_mhz": mhz,
                             "source": iss.get("source")}
        tr = ncu_traffic()
        if tr:
            line["roofline"]["traffic"] = tr.get("bytes_per_launch")
            line["roofline"]["traffic_source"] = tr.get("source")
        print(json.dumps(line), flush=True)
    ctx.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
