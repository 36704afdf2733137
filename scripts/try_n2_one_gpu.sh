# The N > 1 bench step on ONE GPU: 2 (or $1) ranks share GPU 0 over gloo (test hook
# LFE_BENCH_SHARE_GPUS; NCCL refuses duplicate GPUs), with --verify
N=${1:-2}
export LFE_BENCH_SHARE_GPUS=1
for extra in "" "--adaptive 0.75"; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 29511 \
      bench.py --gpus $N --steps 3 --warmup 3 --no-cpu-baseline --verify $extra > gpurun_out/n$N.json 2> gpurun_out/n$N.err
  echo "rc=$?"; python -c "import json; d=json.loads(open('gpurun_out/n$N.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['ms_per_step'], d['verify'], d['config']['parallelism'], d['e2e']['value'])" || tail -20 gpurun_out/n$N.err
done
