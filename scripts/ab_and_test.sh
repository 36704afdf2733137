# inputs abtest/liblfe_{A,B}.so: scripts/ab_build.sh A <git-rev>; scripts/ab_build.sh B
# A/B timing of abtest/liblfe_A.so vs liblfe_B.so (B = the in-tree build) + the fused GPU tests on B
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
bash scripts/ab.sh > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "fused or c1 or c3" > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
