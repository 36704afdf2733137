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

# round 2: peer-halo strips (3 strips in separate allocations, flags signalled), the
# device-resolved adaptive path (DEVT kernel + resolve kernel), lfe_set_stats_device
# on strips, and the orbit-sum statistics kernel on u8 / u16 odd shapes
p = lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02))
with lfe.Context(p) as ctx:
    H, W = img.shape
    cuts = [0, 90, 180, H]
    bufs = [torch.from_numpy(np.ascontiguousarray(img[a:b])).cuda() for a, b in zip(cuts, cuts[1:])]
    outs = [torch.empty_like(x) for x in bufs]
    fl = torch.zeros(3, dtype=torch.int64, device='cuda')
    for k in range(3):
        lfe.lfe_signal(fl[k:k + 1].data_ptr(), 1, torch.cuda.current_stream().cuda_stream)
    for k in range(3):
        above = bufs[k - 1][bufs[k - 1].shape[0] - lfe.LFE_PEER_ROWS:] if k > 0 else None
        below = bufs[k + 1] if k < 2 else None
        ctx.extract_rows_peer(bufs[k], outs[k], above, below,
                              wait_above=fl[k - 1:k].data_ptr() if k > 0 else None,
                              wait_below=fl[k + 1:k + 2].data_ptr() if k < 2 else None, wait_value=1)
    ctx.check()
    print('ok peer strips')
pa = lfe.Params(bit_depth=10, adaptive=lfe.LFE_ADAPT_ZC, zc_threshold=(0.75, 0.75))
with lfe.Context(pa) as ctx:
    d = torch.from_numpy(img).cuda()
    ctx.extract(d)  # device-resolved thresholds, no host sync
    st = torch.zeros(9, dtype=torch.int64, device='cuda')
    ctx.stats_rows(d, 0, 150, 0, 7, lfe.LFE_TOP_IS_EDGE, st)
    ctx.stats_rows(d, 150, 150, 7, 0, lfe.LFE_BOTTOM_IS_EDGE, st)
    ctx.set_stats_device(st)
    out = torch.empty_like(d)
    ctx.extract_rows(d, 0, 300, 0, 0, lfe.LFE_TOP_IS_EDGE | lfe.LFE_BOTTOM_IS_EDGE, out)
    ctx.check()
    print('ok device thresholds')
for bd, shape in [(8, (70, 300)), (16, (133, 1030))]:
    pi = lfe.Params(bit_depth=bd, adaptive=lfe.LFE_ADAPT_ZC, zc_threshold=(0.75, 0.75))
    x = scenes.random_image(np.random.default_rng(bd), *shape, bd, 'mixed')
    with lfe.Context(pi) as ctx:
        st = torch.zeros(9, dtype=torch.int64, device='cuda')
        ctx.stats_rows(torch.from_numpy(x).cuda(), 0, shape[0], 0, 0, 3, st)
        ctx.check()
    print('ok stats5', bd, shape)

# tensor-core LoG (kernel_fused TC / TC12): interior, cheap column edges with warps
# that have no output column (11-bit: they walk; 12-bit: shadow walk), short pieces
rng = np.random.default_rng(5)
for bd, W in ((10, 1444), (11, 2696), (12, 1444), (12, 8192)):
    img = scenes.random_image(rng, 120, W, bd, "mixed")
    for seg in (0, 5):
        with lfe.Context(lfe.Params(bit_depth=bd, zc_threshold=(0.02, 0.02))) as ctx:
            if seg:
                ctx.set_option(lfe.LFE_OPT_TILE_H, seg)
            d = torch.from_numpy(img).cuda()
            out = ctx.extract(d)
            ctx.check()
            print('ok tc', bd, W, seg)
