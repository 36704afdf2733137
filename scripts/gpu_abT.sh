bash scripts/abn.sh "H T" 3
BENCH_ARGS="--config c4" bash scripts/abn.sh "H T" 2
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
