#!/bin/bash
# Persistent launch on/off (debug-knob build, LIFE_PERSIST_FILL=101 disables it).
mkdir -p gpurun_out
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
: > gpurun_out/p_kb.jsonl
for f in 95 101; do
  LIFE_PERSIST_FILL=$f timeout 300 python tools/kbench.py 16384x16384,8192x8192,4096x4096,65536x65536 480 16 | sed "s/^{/{\"fill\": $f, /" >> gpurun_out/p_kb.jsonl
  LIFE_PERSIST_FILL=$f timeout 300 python tools/kbench.py 16384x16384,8192x8192 480 12 | sed "s/^{/{\"fill\": $f, /" >> gpurun_out/p_kb.jsonl
done
cat gpurun_out/p_kb.jsonl
