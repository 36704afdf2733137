set -x
timeout 900 python -m pytest tests -m gpu -q -rs -x -k "peer or signal or bench_ranks or c3_full or strips" > gpurun_out/t_peer.txt 2>&1; tail -5 gpurun_out/t_peer.txt
python scripts/scale_projection.py > gpurun_out/scale_proj.txt 2>&1; head -6 gpurun_out/scale_proj.txt
bash scripts/ab.sh
