# inputs abtest/liblfe_{A,B}.so: scripts/ab_build.sh A <git-rev>; scripts/ab_build.sh B
# A/B timing of two liblfe builds on the same box: abtest/liblfe_A.so vs abtest/liblfe_B.so
for i in 1 2 3; do
  for v in A B; do
    LFE_LIB=$PWD/abtest/liblfe_$v.so python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --no-parity | python -c "import json,sys; d=json.load(sys.stdin); print('$v', d['ms_per_step'], d['roofline']['kernel_ms'])"
  done
done
