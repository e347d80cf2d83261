#!/bin/bash
# Interleaved kernel micro-optimisations: parity, then kbench of the three layouts.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pair.py tests/test_gpu_pair_bands.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r4o_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4o_pytest.log
tail -3 gpurun_out/r4o_pytest.log
for rep in 1 2; do
KB_QUAD=6 timeout 200 python tools/kbench.py 262144x262144,65536x65536,32768x32768 120 0
KB_QUAD=5 timeout 200 python tools/kbench.py 262144x262144,65536x65536 120 0
KB_QUAD=0 KB_PAIR=10 timeout 200 python tools/kbench.py 262144x262144,65536x65536,32768x32768 120 0
done
