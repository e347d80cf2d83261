#!/bin/bash
# kbench of kernel-variant builds (LIFE_GPU_LIB), K = 16 / 12 on several shapes.
mkdir -p gpurun_out
: > gpurun_out/var.jsonl
for rep in 1 2; do
for v in "" _U _F _UF; do
  export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu$v.so
  [ -f $LIFE_GPU_LIB ] || continue
  timeout 300 python tools/kbench.py 16384x16384,8192x8192,65536x65536,65535x65535 480 16 >> gpurun_out/var.jsonl
  timeout 300 python tools/kbench.py 40961x12289,16384x16384 480 12 >> gpurun_out/var.jsonl
done
done
cat gpurun_out/var.jsonl
