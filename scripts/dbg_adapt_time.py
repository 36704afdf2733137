"""Why is the extraction slower with the adaptive threshold?  Time the fused
kernel on c3 at several absolute gap thresholds (incl. the adaptive one)."""
import torch

from paper_1304_3992_b200 import lfe, scenes

img = scenes.scene_c3()
d = torch.from_numpy(img).cuda()
out = torch.empty_like(d)


def timeit(p, n=20):
    with lfe.Context(p) as ctx:
        for _ in range(3):
            ctx.extract(d, out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(n):
            ctx.extract(d, out)
        e1.record()
        torch.cuda.synchronize()
        z = ctx.thresholds()[0]
        return e0.elapsed_time(e1) / n, z, float((out.to(torch.int32) > 0).float().mean())


pa = lfe.Params(bit_depth=10, adaptive=lfe.LFE_ADAPT_ZC, zc_threshold=(0.75, 0.75))
with lfe.Context(pa) as ctx:
    ctx.extract(d, out)
    zt = ctx.thresholds()[0]
    _, F0, _ = ctx.mask(0)
    _, F1, _ = ctx.mask(1)
print("adaptive t", zt, "F", F0, F1)
for thr in [(0.0, 0.0), (0.02, 0.02), ((zt[0] - 0.5) / (2**F0 * 1023), (zt[1] - 0.5) / (2**F1 * 1023)), (0.2, 0.2), (1.0, 1.0)]:
    p = lfe.Params(bit_depth=10, zc_threshold=thr)
    ms, z, frac = timeit(p)
    print(f"thr {thr} -> t {z}: {ms:.4f} ms, output nonzero {frac:.4f}")
