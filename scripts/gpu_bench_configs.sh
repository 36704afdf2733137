# every config's bench line (N=1) + the N>1 share-GPU bench tests
set -x
for c in c3 c1 c2 c4 c5; do
  timeout 900 python bench.py --config $c > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; tail -c 1500 gpurun_out/bench_$c.json; tail -3 gpurun_out/bench_$c.err
done
timeout 1200 python -m pytest tests -m gpu -q -rs -k "bench_ranks" > gpurun_out/t_ranks.txt 2>&1; tail -15 gpurun_out/t_ranks.txt
