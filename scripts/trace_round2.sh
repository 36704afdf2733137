# per-CTA globaltimer trace of the fused kernel at the bench config, then the partition fit
rm -f gpurun_out/trace.txt
LFE_DEBUG_TIMING=$PWD/gpurun_out/trace.txt python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline > /dev/null 2>&1
python scripts/dbg_timeline.py gpurun_out/trace.txt
python scripts/partition_fit.py gpurun_out/trace.txt --paired
