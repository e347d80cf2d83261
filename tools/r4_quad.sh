#!/bin/bash
# Quad-layout prototype (debug library, LIFE_QUAD=1): parity, then depth sweep vs the pair kernel.
mkdir -p gpurun_out
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
LIFE_QUAD=1 timeout 600 python tools/quad_check.py 2>&1 | tail -5
: > gpurun_out/q1_kb.jsonl
KB_PAIR=10 timeout 200 python tools/kbench.py 262144x262144,65536x65536,16384x16384 120 0 >> gpurun_out/q1_kb.jsonl
for d in 3 4 5 6; do
  LIFE_QUAD=1 KB_PAIR=$d timeout 200 python tools/kbench.py 262144x262144,65536x65536,16384x16384 $((d*24)) 0 | sed "s/^{/{\"quad\": 1, /" >> gpurun_out/q1_kb.jsonl
done
cat gpurun_out/q1_kb.jsonl
