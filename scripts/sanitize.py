"""Small runs of both kernels for compute-sanitizer (memcheck / racecheck / synccheck)."""
import sys
import numpy as np
import torch
sys.path.insert(0, '.')
from paper_1304_3992_b200 import lfe, scenes
cases = [(scenes.scene_c1(), lfe.Params(bit_depth=8, zc_threshold=(0.02, 0.02))),
         (scenes.scene_c3(size=1400, height=300), lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02))),
         (scenes.random_image(np.random.default_rng(1), 37, 53, 8), lfe.Params(bit_depth=8))]
for kernel in (lfe.LFE_KERNEL_FUSED, lfe.LFE_KERNEL_STAGED):
    for img, p in cases:
        with lfe.Context(p) as ctx:
            ctx.set_option(lfe.LFE_OPT_KERNEL, kernel)
            H, W = img.shape
            esz = img.dtype.itemsize
            Wp = ((W * esz + 15) // 16) * 16 // esz
            d = torch.zeros((H, Wp), dtype=torch.uint8 if esz == 1 else torch.uint16, device='cuda')[:, :W]
            d.copy_(torch.from_numpy(img))
            out = torch.zeros_like(d)
            try:
                ctx.extract(d, out)
                ctx.check()
                print('ok', kernel, img.shape)
            except lfe.LfeError as e:
                print('skip', kernel, img.shape, e)

# NEXT-1..4 paths: two median levels (fused + staged), adaptive statistics pass,
# float masks and response std sources (staged), multi-band launches (3-D TMA map)
extra = [lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02), median_window2=3),
         lfe.Params(bit_depth=10, adaptive=lfe.LFE_ADAPT_ZC, zc_threshold=(0.75, 0.75)),
         lfe.Params(bit_depth=10, mask_mode=lfe.LFE_MASK_F32, std_source=lfe.LFE_STD_RESPONSE_AT_ZC,
                    std_threshold=(0.01, 0.01), median_window2=5),
         lfe.Params(bit_depth=10, log_size=(9, 3), std_window=7, median_window=7)]
img = scenes.scene_c3(size=1400, height=300)
for p in extra:
    with lfe.Context(p) as ctx:
        d = torch.from_numpy(img).cuda()
        out = ctx.extract(d)
        ctx.check()
        print('ok extra', p.median_window2, p.adaptive, p.mask_mode, p.log_size)
with lfe.Context(lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02))) as ctx:
    b = torch.from_numpy(np.stack([img[:, :1344], img[:, 8:1352], img[:, 40:1384]])).cuda()
    ctx.extract_bands(b)
    ctx.check()
    print('ok bands')
# the 3x3 re-check variant of the fused kernel
with lfe.Context(lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02), std3_threshold=(0.4, 0.4))) as ctx:
    ctx.extract(torch.from_numpy(img).cuda())
    ctx.check()
    print('ok recheck')
