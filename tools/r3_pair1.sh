#!/bin/bash
# Pair-layout kernel: parity, then depth sweep against the plain-layout kernel.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_pair.py -m gpu -x -q -p no:cacheprovider > gpurun_out/p1_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/p1_pytest.log
tail -15 gpurun_out/p1_pytest.log
: > gpurun_out/p1_kb.jsonl
KB_PAIR=0 timeout 200 python tools/kbench.py 262144x262144,65536x65536,16384x16384 160 16 >> gpurun_out/p1_kb.jsonl
for d in 6 8 10 12; do
  KB_PAIR=$d timeout 200 python tools/kbench.py 262144x262144,65536x65536,16384x16384 $((d*20)) 0 >> gpurun_out/p1_kb.jsonl
done
cat gpurun_out/p1_kb.jsonl
