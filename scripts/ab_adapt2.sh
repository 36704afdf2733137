# inputs abtest/liblfe_{A,B}.so: scripts/ab_build.sh A <git-rev>; scripts/ab_build.sh B
# A/B of statistics-pass variants on the adaptive bench; then the adaptive GPU tests on the in-tree build
bash scripts/ab_multi.sh "${V:-A B}" --adaptive 0.75
timeout 900 python -m pytest tests -m gpu -x -q -k "adaptive or stats" > gpurun_out/t.txt 2>&1; tail -2 gpurun_out/t.txt
