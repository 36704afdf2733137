mkdir -p gpurun_out
bash scripts/ncu_quick.sh
ncu -i gpurun_out/prof_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass.csv 2>&1
python scripts/ncu_summary.py gpurun_out/prof_fused.ncu-rep > gpurun_out/ncu_fused_summary.txt 2>&1
head -40 gpurun_out/ncu_fused_summary.txt
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
