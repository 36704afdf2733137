LFE_LIB=$PWD/abtest/liblfe_F.so timeout 150 python -m pytest tests/test_gpu_tc.py -x -q 2>&1 | tail -3
sed -i 's/timeout 150/timeout 90/g' scripts/abn.sh
bash scripts/abn.sh "C F" 3
