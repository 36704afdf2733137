# First run of the tensor-core LoG (TC) fused variant: bench c3 both ways, then the GPU suite.
mkdir -p gpurun_out
timeout 300 python bench.py --no-e2e --no-cpu-baseline --steps 10 > gpurun_out/tc1_bench_tc.json 2> gpurun_out/tc1_bench_tc.err; echo "rc=$?"
tail -c 600 gpurun_out/tc1_bench_tc.err
python - <<'PY'
import json
for f in ["gpurun_out/tc1_bench_tc.json"]:
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, d["ms_per_step"], d["roofline"]["kernel_ms"], d.get("parity"))
    except Exception as e:
        print(f, "no line", e)
PY
timeout 300 python bench.py --no-e2e --no-cpu-baseline --no-parity --steps 10 --log-unit cuda 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('cuda cores', d['ms_per_step'], d['roofline']['kernel_ms'])"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15
