LFE_LIB=$PWD/abtest/liblfe_F.so timeout 600 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
bash scripts/abn.sh "C F" 3
