#!/bin/bash
# Quad layout adopted: parity of every interleaved-layout path, then the default bench.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests/test_gpu_pair_bands.py tests/test_gpu_pair.py tests/test_gpu_bands.py tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r4q_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4q_pytest.log
tail -15 gpurun_out/r4q_pytest.log
timeout 900 python bench.py > gpurun_out/r4q_bench.json 2> gpurun_out/r4q_bench.err; echo "bench rc $?"
cat gpurun_out/r4q_bench.json; tail -3 gpurun_out/r4q_bench.err
