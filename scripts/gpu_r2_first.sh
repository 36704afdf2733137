# round-2 first GPU check on the restored tree: smoke, GPU suite, default bench
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -2 gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -rs -x > gpurun_out/t.txt 2>&1; tail -5 gpurun_out/t.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 600 gpurun_out/bench.json
