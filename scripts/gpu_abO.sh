BENCH_ARGS="--adaptive 0.75" bash scripts/abn.sh "H O" 3
for v in H O; do LFE_LIB=$PWD/abtest/liblfe_$v.so ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/la_$v.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-parity --no-e2e --adaptive 0.75 > /dev/null 2>&1; python scripts/launch_summary.py gpurun_out/la_$v.csv | grep stats; done
