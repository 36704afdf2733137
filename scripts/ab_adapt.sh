# inputs abtest/liblfe_{A,B}.so: scripts/ab_build.sh A <git-rev>; scripts/ab_build.sh B
# A/B of the adaptive-threshold variant (statistics pass + extraction): abtest/liblfe_A.so vs _B.so,
# then the adaptive GPU tests on the in-tree build
for i in 1 2 3; do
  for v in A B; do
    LFE_LIB=$PWD/abtest/liblfe_$v.so python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline --adaptive 0.75 | python -c "import json,sys; d=json.load(sys.stdin); print('$v', d['ms_per_step'], d['roofline']['kernel_ms'])"
  done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "adaptive or stats" > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_adapt.csv \
    python bench.py --steps 3 --warmup 2 --no-cpu-baseline --no-e2e --adaptive 0.75 > /dev/null 2>&1
python scripts/launch_summary.py gpurun_out/launches_adapt.csv adaptive
