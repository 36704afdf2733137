# Session-4 start check: smoke, GPU suite, c3 bench line (one GPU).
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1200 python -m pytest tests -m gpu -q -rs --durations=5 > gpurun_out/gputest_s4.txt 2>&1; tail -12 gpurun_out/gputest_s4.txt
timeout 600 python bench.py > gpurun_out/bench_s4.json 2> gpurun_out/bench_s4.err; tail -c 2500 gpurun_out/bench_s4.json
