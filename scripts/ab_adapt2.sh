bash scripts/ab_multi.sh "A B4 B5" --adaptive 0.75
timeout 900 python -m pytest tests -m gpu -x -q -k "adaptive or stats" > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
