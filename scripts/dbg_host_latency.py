"""Host-side cost of one lfe_extract call (no sync), and the adaptive step's
extraction time, for the liblfe selected by LFE_LIB."""
import time

import torch

from paper_1304_3992_b200 import lfe, scenes

img = scenes.scene_c3()
d = torch.from_numpy(img).cuda()
out = torch.empty_like(d)
with lfe.Context(lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02))) as ctx:
    ctx.extract(d, out)
    torch.cuda.synchronize()
    ts = []
    for _ in range(20):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        ctx.extract(d, out)
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    ts.sort()
    print(f"host time per lfe_extract call: median {1e3 * ts[10]:.3f} ms, min {1e3 * ts[0]:.3f} ms")
