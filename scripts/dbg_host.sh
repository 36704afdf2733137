rm -f gpurun_out/host_timeline.txt
LFE_DEBUG_HOST=gpurun_out/host_timeline.txt PYTHONPATH=. python scripts/e2e_sweep.py
