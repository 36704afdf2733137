# full GPU suite + smoke + the bench lines (default, two-level median, adaptive) on the in-tree build
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1; tail -1 gpurun_out/smoke.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --median2 3 --no-cpu-baseline > gpurun_out/bench_m2.json 2>> gpurun_out/bench.err
python bench.py --adaptive 0.75 --no-cpu-baseline > gpurun_out/bench_adapt.json 2>> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_adapt.csv \
    python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --adaptive 0.75 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_adapt.csv adaptive
tail -c 300 gpurun_out/bench.json
