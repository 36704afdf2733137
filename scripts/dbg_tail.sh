# per-CTA globaltimer timeline of the fused kernel on c3 (LFE_DEBUG_TIMING)
rm -f gpurun_out/timeline.txt
LFE_DEBUG_TIMING=gpurun_out/timeline.txt python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null
python scripts/dbg_timeline.py gpurun_out/timeline.txt
