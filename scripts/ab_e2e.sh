# inputs abtest/liblfe_{A,B}.so: scripts/ab_build.sh A <git-rev>; scripts/ab_build.sh B
# A/B of the end-to-end (host buffers) number: abtest/liblfe_A.so vs _B.so, then the host-path GPU tests
for i in 1 2 3; do
  for v in A B; do
    LFE_LIB=$PWD/abtest/liblfe_$v.so python bench.py --steps 10 --warmup 3 --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print('$v', d['e2e']['value'], d['e2e']['h2d_bytes_per_step'], d['ms_per_step'])"
  done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "host or c5 or stream" > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
