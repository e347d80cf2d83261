#!/bin/bash
# Persistent multi-pass launch: parity + timing.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_bands.py -m gpu -x -q -p no:cacheprovider -k "packed_run" > gpurun_out/g3_pytest_run.log 2>&1; echo "rc $?" >> gpurun_out/g3_pytest_run.log
tail -3 gpurun_out/g3_pytest_run.log
grep -q "rc 0" gpurun_out/g3_pytest_run.log || exit 1
timeout 300 python tools/kbench.py 16384x16384,8192x8192,4096x4096,65536x65536,262144x32768 480 16 > gpurun_out/g3_kb.jsonl
timeout 300 python tools/kbench.py 16384x16384,8192x8192 480 12 >> gpurun_out/g3_kb.jsonl
timeout 300 python tools/kbench.py 16384x16384,8192x8192 480 8 >> gpurun_out/g3_kb.jsonl
cat gpurun_out/g3_kb.jsonl
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g3_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g3_pytest.log
tail -3 gpurun_out/g3_pytest.log
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/g3_bench2.json 2> gpurun_out/g3_bench2.err
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/g3_bench5.json 2> gpurun_out/g3_bench5.err
cut -c1-300 gpurun_out/g3_bench*.json
