#!/bin/bash
mkdir -p gpurun_out
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
: > gpurun_out/g12_kb.jsonl
for w in 0 4 6 0 4; do
  LIFE_BYTE_TB_WPS=$w timeout 120 python tools/kbench.py 16384x16384,32768x16384,4096x4096 96 8 1 | sed "s/^{/{\"wps\": $w, /" >> gpurun_out/g12_kb.jsonl
done
cat gpurun_out/g12_kb.jsonl
