timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
for c in c2 c1; do
  for u in auto cuda tensor; do
  timeout 120 python bench.py --config $c --no-e2e --no-cpu-baseline --log-unit $u 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$c $u', d['ms_per_step'], d['roofline']['kernel_ms'], d.get('parity',{}).get('differing'), d['config'].get('log_unit','')[:14])"
  done
done
bash scripts/sanitize.sh > gpurun_out/sanitize_tc.txt 2>&1; cat gpurun_out/sanitize_tc.txt
