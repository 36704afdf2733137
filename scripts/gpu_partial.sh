set -x
timeout 1500 python -m pytest tests -m gpu -q -rs -x -k "c2 or c4 or fused or strips or bands or c1 or peer or median or intensity" > gpurun_out/t_partial.txt 2>&1; tail -4 gpurun_out/t_partial.txt
for f in 0.3 0.45 0.6 1.0; do
  for c in c2 c4; do
    LFE_DEBUG_PARTIAL=$f python bench.py --config $c --no-e2e --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.load(sys.stdin); print('$f $c', d['ms_per_step'], d['roofline']['kernel_ms'])"
  done
done
python bench.py --no-e2e --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.load(sys.stdin); print('c3', d['ms_per_step'], d['roofline']['kernel_ms'])"
