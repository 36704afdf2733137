# ncu --set full of the fused kernel + source page, the launch list, then the bench line (reads the new issue.json only after it is regenerated here)
set -x
bash scripts/ncu_quick.sh
ncu -i gpurun_out/prof_fused.ncu-rep --page source --csv --print-source sass > gpurun_out/src_sass.csv 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
python scripts/ncu_issue.py gpurun_out/prof_fused.ncu-rep "r01 session 2 final (one-op ZC sign flags)" > /dev/null
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --median2 3 --no-cpu-baseline > gpurun_out/bench_m2.json 2>> gpurun_out/bench.err
python bench.py --adaptive 0.75 --no-cpu-baseline > gpurun_out/bench_adapt.json 2>> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>> gpurun_out/bench.err
cp profiles/issue.json gpurun_out/issue.json
tail -c 400 gpurun_out/bench.json
