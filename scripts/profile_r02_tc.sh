# Round-2 measurement bundle with the tensor-core LoG (one GPU); final state of the round.  Outputs in gpurun_out/ (copied to profiles/ by hand).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/gputest.txt 2>&1; tail -3 gpurun_out/gputest.txt
# ncu --set full of the fused kernel (+ source page) -> hash-stamped issue.json / traffic.json
bash scripts/ncu_quick.sh
ncu -i gpurun_out/prof_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass.csv 2>&1
python scripts/ncu_issue.py gpurun_out/prof_fused.ncu-rep "r02 tensor-core LoG (final)" > /dev/null
cp profiles/issue.json profiles/traffic.json gpurun_out/
python scripts/ncu_summary.py gpurun_out/prof_fused.ncu-rep > gpurun_out/ncu_fused_summary.txt 2>&1
bash scripts/ncu_stats.sh
python scripts/ncu_summary.py gpurun_out/prof_stats.ncu-rep > gpurun_out/ncu_stats_summary.txt 2>&1
# launch lists (default and adaptive bench commands)
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity --no-e2e > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_adapt.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity --no-e2e --adaptive 0.75 > /dev/null 2>&1
# bench lines: every config, then the variants
rm -f gpurun_out/bench_configs.jsonl gpurun_out/bench_variants.jsonl
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json >> gpurun_out/bench_configs.jsonl
for c in c1 c2 c4 c5; do python bench.py --config $c >> gpurun_out/bench_configs.jsonl 2>> gpurun_out/bench.err; done
python bench.py --median2 3 --no-cpu-baseline >> gpurun_out/bench_variants.jsonl 2>> gpurun_out/bench.err
python bench.py --log-unit cuda --no-cpu-baseline >> gpurun_out/bench_variants.jsonl 2>> gpurun_out/bench.err
python bench.py --adaptive 0.75 --no-cpu-baseline >> gpurun_out/bench_variants.jsonl 2>> gpurun_out/bench.err
python bench.py --std intensity --no-cpu-baseline >> gpurun_out/bench_variants.jsonl 2>> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 >> gpurun_out/bench_variants.jsonl 2>> gpurun_out/bench.err
# N > 1 step on this one GPU (ranks folded over gloo, peer halos through CUDA IPC): a check, not a measurement
for h in peer nccl; do
  LFE_BENCH_SHARE_GPUS=1 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 \
    --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 --halo $h --verify --no-e2e 2>> gpurun_out/bench.err \
    | tail -1 >> gpurun_out/bench_n2_one_gpu.jsonl
done
python scripts/scale_projection.py > gpurun_out/scale_proj.txt 2>&1
rm -f gpurun_out/host_timeline.txt
python - <<'PY'
import os, sys, time, torch
sys.path.insert(0, '.')
os.environ['LFE_DEBUG_HOST'] = 'gpurun_out/host_timeline.txt'
from paper_1304_3992_b200 import lfe, scenes
img = scenes.scene_c3(); H, W = img.shape
h_in = torch.from_numpy(img).pin_memory(); h_out = torch.empty((H, W), dtype=torch.uint16).pin_memory()
with lfe.Context(lfe.Params(bit_depth=10, zc_threshold=(0.02, 0.02))) as ctx:
    ctx.set_option(lfe.LFE_OPT_HOST_STRIP_ROWS, 1024)
    for _ in range(3): ctx.extract_host_ptr(h_in.data_ptr(), W * 2, W, H, h_out.data_ptr(), W * 2)
PY
python scripts/host_timeline_summary.py gpurun_out/host_timeline.txt 292704000 288000000 > gpurun_out/host_timeline_summary.txt 2>&1
cat gpurun_out/host_timeline_summary.txt
tail -c 300 gpurun_out/bench.json
