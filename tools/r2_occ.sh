#!/bin/bash
# Occupancy sweep: warps per SM of the packed pass kernels (debug-knob build).
mkdir -p gpurun_out
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
S=16384x16384,8192x8192,65536x65536,40961x12289
for d in 16 12 8; do
 for w in 0 6 4; do
  LIFE_FAST_WPB=$w LIFE_WPB=$w LIFE_FAST_BPS=1 timeout 300 python tools/kbench.py $S 480 $d | sed "s/^/{\"wpb\": $w, /; s/{\"wpb\": $w, {/{\"wpb\": $w, /" >> gpurun_out/occ.jsonl
 done
done
cat gpurun_out/occ.jsonl
