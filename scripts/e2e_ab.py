"""A/B of lfe_extract_host end-to-end time on c3 (abtest/liblfe_{A,B}.so) vs strip size."""
import os
import subprocess
import sys

code = r'''
import sys, time, torch
sys.path.insert(0, ".")
from paper_1304_3992_b200 import lfe, scenes
img = scenes.scene_c3()
H, W = img.shape
h_in = torch.from_numpy(img).pin_memory()
h_out = torch.empty((H, W), dtype=torch.uint16).pin_memory()
with lfe.Context(lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02))) as ctx:
    for S in (768, 1024, 1536, 2048):
        ctx.set_option(lfe.LFE_OPT_HOST_STRIP_ROWS, S)
        ctx.extract_host_ptr(h_in.data_ptr(), W * 2, W, H, h_out.data_ptr(), W * 2)
        ts = []
        for _ in range(8):
            t0 = time.perf_counter()
            ctx.extract_host_ptr(h_in.data_ptr(), W * 2, W, H, h_out.data_ptr(), W * 2)
            ts.append(time.perf_counter() - t0)
        ts.sort()
        print(sys.argv[1], S, "median %.3f ms best %.3f ms" % (1e3 * ts[len(ts) // 2], 1e3 * ts[0]))
'''
for v in ("A", "B", "A", "B"):
    env = dict(os.environ, LFE_LIB=os.path.abspath(f"abtest/liblfe_{v}.so"))
    print(subprocess.run([sys.executable, "-c", code, v], env=env, capture_output=True, text=True).stdout, end="")
