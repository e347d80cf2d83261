#!/bin/bash
mkdir -p gpurun_out
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
: > gpurun_out/p2_kb.jsonl
for m in 0 8 9 1; do
  LIFE_PERSIST_MODE=$m timeout 300 python tools/kbench.py 16384x16384,8192x8192 480 16 | sed "s/^{/{\"mode\": $m, /" >> gpurun_out/p2_kb.jsonl
done
LIFE_PERSIST_FILL=101 timeout 300 python tools/kbench.py 16384x16384,8192x8192 480 16 | sed "s/^{/{\"mode\": \"off\", /" >> gpurun_out/p2_kb.jsonl
cat gpurun_out/p2_kb.jsonl
