# inputs abtest/liblfe_{A,B}.so: scripts/ab_build.sh A <git-rev>; scripts/ab_build.sh B
# A/B timing of abtest/liblfe_A.so vs abtest/liblfe_B.so, then the FULL GPU suite on the in-tree build
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash scripts/ab.sh > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -5 gpurun_out/t.txt
if [ -x abtest/ubench ]; then abtest/ubench > gpurun_out/ubench.txt 2>&1; tail -8 gpurun_out/ubench.txt; fi
