"""lfe_extract_host end-to-end time on c3 vs the host strip size (pinned buffers)."""
import time

import numpy as np
import torch

from paper_1304_3992_b200 import lfe, scenes

img = scenes.scene_c3()
H, W = img.shape
h_in = torch.from_numpy(img).pin_memory()
h_out = torch.empty((H, W), dtype=torch.uint16).pin_memory()
with lfe.Context(lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02))) as ctx:
    for S in (128, 256, 512, 1024, 2048, 4096):
        ctx.set_option(lfe.LFE_OPT_HOST_STRIP_ROWS, S)
        ctx.extract_host_ptr(h_in.data_ptr(), W * 2, W, H, h_out.data_ptr(), W * 2)
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            ctx.extract_host_ptr(h_in.data_ptr(), W * 2, W, H, h_out.data_ptr(), W * 2)
            ts.append(time.perf_counter() - t0)
        t = min(ts)
        print(f"strip {S:5d}: {1e3 * t:.3f} ms  {H * W / t / 1e9:.2f} Gpx/s")
