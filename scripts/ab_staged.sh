# inputs abtest/liblfe_{A,B}.so: scripts/ab_build.sh A <git-rev>; scripts/ab_build.sh B
# A/B of the general (staged) kernel on c3 + its parity tests on B
for v in A B; do
  LFE_LIB=$PWD/abtest/liblfe_$v.so python bench.py --kernel staged --steps 5 --warmup 3 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print('$v staged', d['ms_per_step'])"
done
PYTHONPATH=. timeout 900 python -m pytest tests -m gpu -q -x -k "sweep or tile or f32 or response or adaptive or two_level or strips or bands" 2>&1 | tail -2
