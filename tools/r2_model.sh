#!/bin/bash
# Segment cost model change: base vs new library on the config shapes.
: > gpurun_out/g20_kb.jsonl
for lib in liblife_gpu_base.so liblife_gpu.so liblife_gpu_base.so liblife_gpu.so; do
  LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/$lib timeout 200 python tools/kbench.py 65536x65536,262144x65536,16384x16384,40961x12289,8192x8192,32768x16384,131072x65536,65535x65535 160 0 >> gpurun_out/g20_kb.jsonl
done
cat gpurun_out/g20_kb.jsonl
