import sys, numpy as np, torch
sys.path.insert(0, '.')
import oracle as O
from paper_1304_3992_b200 import lfe, scenes
def run(img, p, kernel):
    with lfe.Context(p) as ctx:
        ctx.set_option(lfe.LFE_OPT_KERNEL, kernel)
        d = torch.from_numpy(img).cuda()
        out = ctx.extract(d)
        st = ctx.last_async_error()
        return out.cpu().numpy(), st
for bd, img in [(10, scenes.scene_c3(size=600, height=300)), (8, scenes.scene_c1())]:
    p = lfe.Params(bit_depth=bd, zc_threshold=(0.02, 0.02))
    op = O.Params(bit_depth=bd, zc_threshold=(0.02, 0.02))
    want = O.run(img, op)
    got, st = run(img, p, lfe.LFE_KERNEL_FUSED)
    bad = np.argwhere(got != want)
    print(bd, 'status', st, 'bad', len(bad), bad[:5].tolist(), flush=True)
    if len(bad):
        y, x = bad[0]; print(got[y, x-3:x+4], want[y, x-3:x+4])
