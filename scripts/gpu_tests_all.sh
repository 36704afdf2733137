# GPU suite without -x (every failure listed), with durations
set -x
timeout 2400 python -m pytest tests -m gpu -q -rs --durations=15 > gpurun_out/t_all.txt 2>&1; tail -40 gpurun_out/t_all.txt
