# full GPU suite + smoke + a few bench lines
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=10 > gpurun_out/t_all.txt 2>&1; tail -16 gpurun_out/t_all.txt
python bench.py --adaptive 0.75 --no-cpu-baseline > gpurun_out/bench_adapt.json 2> gpurun_out/bench_adapt.err; tail -c 300 gpurun_out/bench_adapt.json
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; tail -c 300 gpurun_out/bench.json
