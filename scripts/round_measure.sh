# Round measurement bundle (one GPU): full GPU suite + smoke, the default bench line,
# variant bench lines (two-level median, adaptive), the ncu launch list of the default
# command, and one ncu --set full capture of the fused kernel.  Outputs in gpurun_out/.
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks.mem --format=csv > gpurun_out/gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --median2 3 --no-cpu-baseline > gpurun_out/bench_m2.json 2>> gpurun_out/bench.err
python bench.py --adaptive 0.75 --no-cpu-baseline > gpurun_out/bench_adapt.json 2>> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:fused_kernel -s 3 -c 1 -o gpurun_out/prof_fused -f \
    python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_full.log 2>&1
tail -c 400 gpurun_out/bench.json
