BENCH_ARGS="--log-unit cuda" bash scripts/abn.sh "P H" 2
