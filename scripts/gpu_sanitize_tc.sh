mkdir -p gpurun_out
bash scripts/sanitize.sh > gpurun_out/sanitize_tc.txt 2>&1
cat gpurun_out/sanitize_tc.txt
