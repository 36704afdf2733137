# peer-halo path: new GPU tests (in-process strips, validation, IPC bench ranks), then the whole suite
set -x
timeout 900 python -m pytest tests -m gpu -q -rs -x -k "peer or signal or bench_ranks" > gpurun_out/t_peer.txt 2>&1; tail -30 gpurun_out/t_peer.txt
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/t_all.txt 2>&1; tail -5 gpurun_out/t_all.txt
timeout 600 python bench.py --no-e2e > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; tail -c 300 gpurun_out/bench_c3.json
