LFE_LIB=$PWD/abtest/liblfe_R.so timeout 300 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -2
bash scripts/abn.sh "H R" 3
