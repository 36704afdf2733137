set -x
timeout 1500 python -m pytest tests -m gpu -q -rs -x -k "fused or strips or peer or c3_full or c1 or c2 or median or bands or recheck or bench_ranks" > gpurun_out/t_phase.txt 2>&1; tail -4 gpurun_out/t_phase.txt
bash scripts/ab.sh
python scripts/scale_projection.py > gpurun_out/scale_proj.txt 2>&1; head -6 gpurun_out/scale_proj.txt
for c in c1 c2 c4; do python bench.py --config $c --no-e2e --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.load(sys.stdin); print('$c', d['ms_per_step'], d['roofline']['kernel_ms'])"; done
