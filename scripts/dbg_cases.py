import sys, subprocess
code = r'''
import sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_1304_3992_b200 import lfe
bd, H, W, hm, mask = [int(v) for v in sys.argv[1:6]]
dt = np.uint8 if bd <= 8 else np.uint16
img = (np.random.default_rng(0).integers(0, 1 << bd, (H, W))).astype(dt)
p = lfe.Params(bit_depth=bd, zc_threshold=(0.02, 0.02), hybrid_median=bool(hm), out_mode=mask)
with lfe.Context(p) as ctx:
    ctx.set_option(lfe.LFE_OPT_KERNEL, lfe.LFE_KERNEL_FUSED)
    out = ctx.extract(torch.from_numpy(img).cuda())
    print('status', ctx.last_async_error())
'''
for case in ["10 300 600 1 0", "10 512 512 1 0", "8 512 512 1 0", "8 300 600 1 0", "8 300 4096 1 0",
             "8 300 600 0 0", "8 300 600 1 1", "10 300 600 1 1", "8 300 600 0 1", "12 100 100 1 0"]:
    r = subprocess.run([sys.executable, '-c', code] + case.split(), capture_output=True, text=True)
    print(case, '->', (r.stdout.strip() or r.stderr.strip().splitlines()[-1])[:120], flush=True)
