mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -5
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
for v in "" "--median2 3" "--adaptive 0.75" "--config c5"; do
  timeout 300 python bench.py --no-e2e --no-cpu-baseline $v 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['kernel_ms'], d.get('parity'))"
done
