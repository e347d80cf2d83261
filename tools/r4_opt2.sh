#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pair.py tests/test_gpu_pair_bands.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r4o_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4o_pytest.log
tail -3 gpurun_out/r4o_pytest.log
for rep in 1 2; do
KB_QUAD=7 timeout 200 python tools/kbench.py 262144x262144,65536x65536,32768x32768,131072x8192 126 0
KB_QUAD=6 timeout 200 python tools/kbench.py 262144x262144,65536x65536,32768x32768,131072x8192 120 0
done
