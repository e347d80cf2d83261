#!/bin/bash
mkdir -p gpurun_out
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
: > gpurun_out/occ2.jsonl
for w in 0 4 0 4; do
  LIFE_FAST_WPB=$w LIFE_FAST_BPS=1 timeout 300 python tools/kbench.py 16384x16384,8192x8192,32768x16384 480 16 | sed "s/^{/{\"wpb\": $w, /" >> gpurun_out/occ2.jsonl
done
cat gpurun_out/occ2.jsonl
