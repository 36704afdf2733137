bash scripts/abn.sh "H M" 4
BENCH_ARGS="--config c5" bash scripts/abn.sh "H M" 1
BENCH_ARGS="--config c4" bash scripts/abn.sh "H M" 1
