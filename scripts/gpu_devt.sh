set -x
timeout 1200 python -m pytest tests -m gpu -q -rs -x -k "adaptive or stats or resolve or bench_ranks" > gpurun_out/t_devt.txt 2>&1; tail -5 gpurun_out/t_devt.txt
for i in 1 2; do python bench.py --adaptive 0.75 --no-e2e --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.load(sys.stdin); print('adaptive', d['ms_per_step'], d['roofline']['kernel_ms'], d['gpu_launches'])"; done
