#!/bin/bash
# AddressSanitizer + UndefinedBehaviorSanitizer builds of the CPU oracle and of
# liblfe's host core (lfe_host.cu + the test entries; the kernel objects of the
# normal build are linked uninstrumented), then the oracle pins and the ABI tests
# run against them in a python that preloads the sanitizer runtimes.  CPU only.
#   scripts/sanitize_host.sh [pytest -k expression for the oracle pins]
set -euo pipefail
cd "$(dirname "$0")/.."
OUT=${SAN_OUT:-/tmp/lfe_san}
mkdir -p "$OUT"
SAN="-fsanitize=address,undefined -fno-sanitize-recover=undefined -fno-omit-frame-pointer"
python -c "import __graft_entry__ as g; g.build()" > /dev/null
gcc -O1 -g -std=c11 -fopenmp -fPIC -shared $SAN oracle/lfe_oracle.c -o "$OUT/liblfe_oracle_san.so" -lm
NV="nvcc -gencode arch=compute_100a,code=sm_100a -O1 -g -std=c++17 -I include -I paper_1304_3992_b200/csrc"
$NV -Xcompiler -fPIC,-fsanitize=address,-fsanitize=undefined,-fno-sanitize-recover=undefined,-fno-omit-frame-pointer \
    -c paper_1304_3992_b200/csrc/lfe_host.cu -o "$OUT/lfe_host_san.o"
$NV -Xcompiler -fPIC,-fsanitize=address,-fsanitize=undefined,-fno-sanitize-recover=undefined,-fno-omit-frame-pointer \
    -c paper_1304_3992_b200/csrc/test/lfe_test.cu -o "$OUT/lfe_test_san.o"
OBJS=$(ls paper_1304_3992_b200/build/*.o | grep -v -e lfe_host.o -e lfe_test.o)
$NV -shared -Xcompiler -fsanitize=address,-fsanitize=undefined -o "$OUT/liblfe.so" "$OUT/lfe_host_san.o" $OBJS
$NV -shared -Xcompiler -fsanitize=address,-fsanitize=undefined -o "$OUT/liblfe_test.so" "$OUT/lfe_test_san.o" \
    -L "$OUT" -llfe -Xlinker -rpath,"$OUT"
PRE="$(gcc -print-file-name=libasan.so):$(gcc -print-file-name=libubsan.so)"
export ASAN_OPTIONS=detect_leaks=0:abort_on_error=1 UBSAN_OPTIONS=print_stacktrace=1:halt_on_error=1
LD_PRELOAD="$PRE" LFE_ORACLE_LIB="$OUT/liblfe_oracle_san.so" \
    python -m pytest tests/test_oracle_pins.py tests/test_oracle_properties.py tests/test_median_networks.py \
    -q -x -p no:cacheprovider -k "${1:-not nothing}"
LD_PRELOAD="$PRE" LFE_LIB="$OUT/liblfe.so" LFE_TEST_LIB="$OUT/liblfe_test.so" \
    python -m pytest tests/test_abi_cpu.py -q -x -p no:cacheprovider
echo "sanitizers: clean"
