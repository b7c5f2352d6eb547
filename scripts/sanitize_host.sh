#!/usr/bin/env bash
# AddressSanitizer + UndefinedBehaviorSanitizer builds of the host code, run on the CPU test suite
# (no GPU needed): the oracle (oracle/hc_oracle.c) and the host side of libhc.so (the system
# compiler and the C ABI, csrc/host/*.cpp; the kernels are compiled as usual).  Logs go to
# gpurun_out/asan_*.log (copy them to profiles/ to keep them).
set -u
mkdir -p gpurun_out /tmp/hc_asan
ASAN=$(gcc -print-file-name=libasan.so)
UBSAN=$(gcc -print-file-name=libubsan.so)
gcc -std=gnu99 -O1 -g -fPIC -shared -ffp-contract=off -fno-fast-math -fsanitize=address,undefined \
    -fno-omit-frame-pointer -o /tmp/hc_asan/liboracle.so oracle/hc_oracle.c -lm -lpthread
HCB_VARIANT=asan HCB_DEFINES="HCB_ASAN_BUILD=1" HCB_HOST_FLAGS="-fsanitize=address -fsanitize=undefined -fno-omit-frame-pointer" \
    python paper_2112_03444_b200/build.py > /dev/null
export ASAN_OPTIONS=detect_leaks=0:halt_on_error=1:verify_asan_link_order=0
export UBSAN_OPTIONS=halt_on_error=1:print_stacktrace=1
ORACLE_SO=/tmp/hc_asan/liboracle.so LD_PRELOAD="$ASAN $UBSAN" timeout 1800 python -m pytest tests/test_oracle_pins.py -q -x \
    > gpurun_out/asan_oracle.log 2>&1; echo "oracle (ASan+UBSan): $(tail -1 gpurun_out/asan_oracle.log)"
HC_LIB_PATH=paper_2112_03444_b200/lib_asan/libhc.so LD_PRELOAD="$ASAN $UBSAN" timeout 1800 python -m pytest tests/test_abi_cpu.py -q -x \
    > gpurun_out/asan_host.log 2>&1; echo "libhc host (ASan+UBSan): $(tail -1 gpurun_out/asan_host.log)"
