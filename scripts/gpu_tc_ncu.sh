# ncu --set full of the TC fused kernel at the c3 bench config, plus its source page
mkdir -p gpurun_out
bash scripts/ncu_quick.sh
ncu -i gpurun_out/prof_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass.csv 2>&1
python scripts/ncu_summary.py gpurun_out/prof_fused.ncu-rep > gpurun_out/ncu_fused_summary.txt 2>&1
head -60 gpurun_out/ncu_fused_summary.txt
