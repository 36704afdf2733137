# inputs abtest/liblfe_{A,B}.so: scripts/ab_build.sh A <git-rev>; scripts/ab_build.sh B
# A/B timing (abtest/liblfe_A.so vs abtest/liblfe_B.so) + GPU tests of the fused path + one ncu
# --set full capture of the in-tree build's fused kernel (source page for scripts/ncu_lines.py)
set -x
bash scripts/ab.sh > gpurun_out/ab.txt 2>&1
cat gpurun_out/ab.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/t.txt 2>&1; tail -3 gpurun_out/t.txt
bash scripts/ncu_quick.sh
ncu -i gpurun_out/prof_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass.csv 2>&1
