BENCH_ARGS="--config c2" bash scripts/abn.sh "M M2" 3
