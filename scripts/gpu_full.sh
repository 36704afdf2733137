# full GPU test suite + smoke + bench (default and the two-level median variant)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -3 gpurun_out/smoke.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -5 gpurun_out/t.txt
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json
timeout 600 python bench.py --steps 20 --warmup 5 --median2 3 --no-cpu-baseline > gpurun_out/bench_m2.json 2>> gpurun_out/bench.err; cat gpurun_out/bench_m2.json
