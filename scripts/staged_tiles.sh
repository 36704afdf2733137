# general-kernel tile sweep on c3 (tile shape never changes the result)
for t in 64x32 128x32 64x64 128x16 256x16 128x64 96x48; do
  python bench.py --kernel staged --tile $t --steps 5 --warmup 2 --no-e2e --no-cpu-baseline | python -c "import json,sys; d=json.load(sys.stdin); print('$t', d['ms_per_step'])"
done
