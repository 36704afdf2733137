BENCH_ARGS="--adaptive 0.75" bash scripts/abn.sh "H S" 3
LFE_LIB=$PWD/abtest/liblfe_S.so timeout 600 python -m pytest tests -m gpu -x -q -k "adaptive or stats" 2>&1 | tail -3
LFE_LIB=$PWD/abtest/liblfe_S.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_adapt_S.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity --no-e2e --adaptive 0.75 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_adapt_S.csv | grep stats
