timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
for c in c4 c3; do
  timeout 120 python bench.py --config $c --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c', d['ms_per_step'], d['roofline']['kernel_ms'], d.get('parity',{}).get('differing'), d['config'].get('log_unit','')[:14])"
done
timeout 120 python bench.py --config c4 --no-e2e --no-cpu-baseline --no-parity --log-unit cuda 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('c4 cuda', d['ms_per_step'], d['roofline']['kernel_ms'])"
