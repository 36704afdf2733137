# ncu --set full of one statistics-pass launch (adaptive bench config)
mkdir -p gpurun_out
ncu --set full --clock-control none -k regex:stats -s 2 -c 1 -o gpurun_out/prof_stats -f \
    python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu-baseline --adaptive 0.75 --no-parity > gpurun_out/ncu_stats.log 2>&1
tail -2 gpurun_out/ncu_stats.log | cut -c1-200
