import sys; sys.path.insert(0, '.')
import numpy as np, torch
import oracle as O
from paper_1304_3992_b200 import lfe, scenes
sys.path.insert(0, 'tests')
p = lfe.Params(bit_depth=8, adaptive=lfe.LFE_ADAPT_ZC, zc_threshold=(0.75, 0.75))
rng = np.random.default_rng(400)
for (H, W) in [(1, 17), (5, 40), (64, 200)]:
    img = scenes.random_image(rng, H, W, 8, "mixed")
    Wp = ((W + 15) // 16) * 16 + 16
    d = torch.zeros((H, Wp), dtype=torch.uint8, device="cuda")[:, :W]
    d.copy_(torch.from_numpy(img))
    with lfe.Context(p) as ctx:
        st = torch.zeros(9, dtype=torch.int64, device="cuda")
        ctx.stats_rows(d, 0, H, 0, 0, 3, st)
        v = [int(x) for x in st.cpu()]
        ctx.set_stats(v)
        zh = ctx.thresholds()[0]
        zd = ctx.test_resolve(v)
        out_h = torch.zeros((H, Wp), dtype=torch.uint8, device="cuda")[:, :W]; ctx.extract_rows(d, 0, H, 0, 0, 3, out_h); ctx.check()
        ctx.set_stats_device(st)
        out_d = torch.zeros((H, Wp), dtype=torch.uint8, device="cuda")[:, :W]; ctx.extract_rows(d, 0, H, 0, 0, 3, out_d); ctx.check()
        out_e = torch.zeros((H, Wp), dtype=torch.uint8, device="cuda")[:, :W]; ctx.extract(d, out_e); ctx.check()
    want = O.run(img, O.Params(bit_depth=8, adaptive=1, zc_threshold=(0.75, 0.75)))
    print(H, W, v, zh, zd, (out_h.cpu().numpy() != want).sum(), (out_d.cpu().numpy() != want).sum(), (out_e.cpu().numpy() != want).sum())

# the exact GPU-test sequence
sys.path.insert(0, 'tests')
import test_gpu_parity as T
lfe.load()
p = list(T._adaptive_cases())[0]
rng = np.random.default_rng(400)
import itertools
for (H, W), kind in itertools.product(T.SHAPES + [(129, 463)], ["mixed", "blocks"]):
    img = scenes.random_image(rng, H, W, p.bit_depth, kind)
    got = T.run_gpu(img, p, lfe.LFE_KERNEL_AUTO)
    want = O.run(img, T._oparams(p))
    print(H, W, kind, int((got != want).sum()))
