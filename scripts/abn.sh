# A/B/... timing of liblfe builds abtest/liblfe_<V>.so on one box (c3 bench config unless BENCH_ARGS)
# usage: scripts/abn.sh "A B C" [rounds]
vs=${1:-"A B"}; n=${2:-3}
for v in $vs; do
  LFE_LIB=$PWD/abtest/liblfe_$v.so timeout 150 python bench.py --steps 10 --warmup 3 --no-e2e --no-cpu-baseline $BENCH_ARGS 2>/dev/null \
    | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v parity', d.get('parity',{}).get('differing'), d['roofline']['kernel_ms'])"
done
for i in $(seq $n); do
  for v in $vs; do
    LFE_LIB=$PWD/abtest/liblfe_$v.so timeout 150 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-parity $BENCH_ARGS 2>/dev/null \
      | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', d['ms_per_step'], d['roofline']['kernel_ms'])"
  done
done
