# run a subset of GPU tests: $1 = pytest -k expression
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/t.txt 2>&1
tail -30 gpurun_out/t.txt
