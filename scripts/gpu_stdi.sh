set -x
timeout 1500 python -m pytest tests -m gpu -q -rs -x -k "intensity" > gpurun_out/t_stdi.txt 2>&1; tail -15 gpurun_out/t_stdi.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/t_all.txt 2>&1; tail -4 gpurun_out/t_all.txt
python - <<'PY'
import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_1304_3992_b200 import lfe, scenes
img = torch.from_numpy(scenes.scene_c3()).cuda()
for k, name in [(lfe.LFE_KERNEL_FUSED, 'fused'), (lfe.LFE_KERNEL_STAGED, 'staged')]:
    p = lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02), std_source=lfe.LFE_STD_INTENSITY, std_threshold=(20.0, 20.0))
    with lfe.Context(p) as ctx:
        ctx.set_option(lfe.LFE_OPT_KERNEL, k)
        out = torch.empty_like(img)
        for _ in range(3): ctx.extract(img, out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): ctx.extract(img, out)
        e1.record(); torch.cuda.synchronize()
        print('intensity std c3', name, e0.elapsed_time(e1) / 10, 'ms')
PY
