set -x
timeout 900 python -m pytest tests -m gpu -q -rs -x -k "stats or adaptive" > gpurun_out/t_stats.txt 2>&1; tail -5 gpurun_out/t_stats.txt
for i in 1 2; do
  python bench.py --adaptive 0.75 --no-e2e --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.load(sys.stdin); print('orbit', d['ms_per_step'], d['roofline']['kernel_ms'])"
  LFE_STATS_GENERIC=1 python bench.py --adaptive 0.75 --no-e2e --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.load(sys.stdin); print('generic', d['ms_per_step'], d['roofline']['kernel_ms'])"
done
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_adapt.csv \
    python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --no-parity --adaptive 0.75 > /dev/null 2>&1
grep -i stats gpurun_out/launches_adapt.csv | tail -3
