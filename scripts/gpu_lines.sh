# the per-config and variant bench lines only (same commands as the bundle)
mkdir -p gpurun_out
rm -f gpurun_out/bench_configs.jsonl gpurun_out/bench_variants.jsonl
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; cat gpurun_out/bench.json >> gpurun_out/bench_configs.jsonl
for c in c1 c2 c4 c5; do python bench.py --config $c >> gpurun_out/bench_configs.jsonl 2>> gpurun_out/bench.err; done
python bench.py --median2 3 --no-cpu-baseline >> gpurun_out/bench_variants.jsonl 2>> gpurun_out/bench.err
python bench.py --log-unit cuda --no-cpu-baseline >> gpurun_out/bench_variants.jsonl 2>> gpurun_out/bench.err
python bench.py --adaptive 0.75 --no-cpu-baseline >> gpurun_out/bench_variants.jsonl 2>> gpurun_out/bench.err
python bench.py --std intensity --no-cpu-baseline >> gpurun_out/bench_variants.jsonl 2>> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 >> gpurun_out/bench_variants.jsonl 2>> gpurun_out/bench.err
