# Round-2 measurement bundle (one GPU): ncu --set full of the fused kernel (+ source page),
# issue.json / traffic.json stamped with the kernel-source hash, the launch list of the
# default bench command, then the bench lines (default, two-level median, adaptive, reference).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
bash scripts/ncu_quick.sh
ncu -i gpurun_out/prof_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass.csv 2>&1
python scripts/ncu_issue.py gpurun_out/prof_fused.ncu-rep "r02" > /dev/null
cp profiles/issue.json profiles/traffic.json gpurun_out/
python scripts/ncu_summary.py gpurun_out/prof_fused.ncu-rep > gpurun_out/ncu_fused_summary.txt 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity > /dev/null 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --median2 3 --no-cpu-baseline > gpurun_out/bench_m2.json 2>> gpurun_out/bench.err
python bench.py --adaptive 0.75 --no-cpu-baseline > gpurun_out/bench_adapt.json 2>> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
tail -c 400 gpurun_out/bench.json
