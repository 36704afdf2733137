set -x
timeout 900 python -m pytest tests -m gpu -q -rs -x -k "peer or signal or bench_ranks or c3_full" > gpurun_out/t_peer.txt 2>&1; tail -5 gpurun_out/t_peer.txt
bash scripts/ab.sh
