"""One-GPU projection of the strong-scaling curve of the c3 bench step at
N = 1, 2, 4, 8: for every rank k of N, that rank's exact
device work on this GPU -- its row strip of the 12000^2 scene with the halo rows
its neighbours supply -- timed with CUDA events, in two schedules:

  split : the NCCL path of bench.py (interior band while the exchange is in
          flight, then one launch per boundary band) -- exchange time excluded
  single: one lfe_extract_rows launch over the whole strip with its halo rows
  peer  : bench.py's peer-halo step: lfe_signal + one lfe_extract_rows_peer
          launch, the strip in its own allocation and the neighbours' rows read
          in place from two other allocations (on this GPU: HBM, not NVLink)

The projected N-GPU step is the max over ranks; efficiency = T1 / (N * TN).
NVLink transfer and NCCL latency are NOT included (one GPU): a lower bound on
the per-step time, an upper bound on efficiency.

    python scripts/scale_projection.py [--reps 20] [--config c3|c1|c2|c5]
"""
import argparse
import json
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1304_3992_b200 import lfe  # noqa: E402
from paper_1304_3992_b200.shard import StripShard  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--config", default="c3")
    a = ap.parse_args()
    cfg = dict(bench.CFG[a.config])
    H, W = cfg["H"], cfg["W"]
    p = bench.workload_params(cfg)
    sc = bench.Scene(a.config, cfg)
    sc.hold(0, H)
    tdt = torch.uint8 if cfg["bit_depth"] <= 8 else torch.uint16
    esz = 1 if tdt == torch.uint8 else 2
    dev = torch.device("cuda", 0)
    ctx = lfe.Context(p)
    halo = ctx.halo
    img = torch.from_numpy(sc.rows(0, H)).to(dev)
    out = torch.empty_like(img)
    pitch = img.stride(0) * esz
    s = torch.cuda.current_stream().cuda_stream
    rows = []

    def timed(calls):
        for _ in range(3):
            for c in calls:
                c()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.reps):
            for c in calls:
                c()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / a.reps

    def call(r0, n, ha, hb, flags):
        return lambda: lfe.lfe_extract_rows(ctx.handle, img.data_ptr() + r0 * pitch, pitch, W, n, ha, hb, flags,
                                            out.data_ptr() + r0 * pitch, pitch, s)

    flag = torch.zeros(4, dtype=torch.int64, device=dev)

    def peer_call(sh):
        own = img[sh.a:sh.b].clone()
        o = torch.empty_like(own)
        above = img[sh.a - halo:sh.a].clone() if sh.rank > 0 else None
        below = img[sh.b:sh.b + halo].clone() if sh.rank < sh.world - 1 else None
        keep.append((own, o, above, below))
        cnt = [0]

        def f():
            cnt[0] += 1
            lfe.lfe_signal(flag[0:1].data_ptr(), cnt[0], s)
            lfe.lfe_extract_rows_peer(ctx.handle, own.data_ptr(), pitch, W, sh.rows,
                                      above.data_ptr() if above is not None else 0, pitch,
                                      below.data_ptr() if below is not None else 0, pitch, sh.edge_flags(),
                                      flag[0:1].data_ptr() if above is not None else 0,
                                      flag[0:1].data_ptr() if below is not None else 0, cnt[0],
                                      o.data_ptr(), pitch, s)
        return f

    res = {}
    for N in (1, 2, 4, 8):
        split, single, peer = [], [], []
        for k in range(N):
            keep = []
            sh = StripShard(H, W, k, N, halo)
            calls = [call(sh.a + b[0], b[1], b[2], b[3], b[4]) for b in sh.bands()]
            split.append(timed(calls))
            single.append(timed([call(sh.a, sh.rows, sh.ha, sh.hb, sh.edge_flags())]))
            peer.append(timed([peer_call(sh)]))
        res[N] = (max(split), max(single), max(peer), split, single, peer)
    t1 = res[1][1]
    lines = [f"# scripts/scale_projection.py --config {a.config} --reps {a.reps} (one B200; per-rank device work only,"
             " no NVLink / NCCL time)",
             "N  split_ms  single_ms  peer_ms (max over ranks)  Mpx/s(peer)  eff(split)  eff(single)  eff(peer)"]
    for N, (ms_split, ms_single, ms_peer, *_) in res.items():
        lines.append(f"{N}  {ms_split:.4f}  {ms_single:.4f}  {ms_peer:.4f}  {H * W / ms_peer / 1e3:.0f}  "
                     f"{t1 / (N * ms_split):.3f}  {t1 / (N * ms_single):.3f}  {t1 / (N * ms_peer):.3f}")
    print("\n".join(lines))
    print(json.dumps({str(N): {"split_ms_per_rank": [round(x, 4) for x in v[3]],
                               "single_ms_per_rank": [round(x, 4) for x in v[4]],
                               "peer_ms_per_rank": [round(x, 4) for x in v[5]]} for N, v in res.items()}))


if __name__ == "__main__":
    main()
