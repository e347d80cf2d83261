#!/bin/bash
# Trip-level prefetch in the plain-layout packed kernels: parity suite (not slow), then kbench.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bands.py tests/test_gpu_multi.py tests/test_rule_network.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r4p_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4p_pytest.log
tail -3 gpurun_out/r4p_pytest.log
for rep in 1 2; do
KB_PAIR=0 KB_QUAD=0 timeout 300 python tools/kbench.py 16384x16384,40961x12289,65536x65536,262144x65536,65535x65535,8192x8192 160 16
KB_PAIR=0 KB_QUAD=0 timeout 300 python tools/kbench.py 40961x12289,16384x16384 144 12
done
