#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/g16_kb.jsonl
for lib in liblife_gpu_base.so liblife_gpu.so liblife_gpu_base.so liblife_gpu.so; do
  LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/$lib timeout 120 python tools/kbench.py 8192x8192,4096x4096,6144x6144,16384x16384,2048x2048 480 16 >> gpurun_out/g16_kb.jsonl
  LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/$lib timeout 120 python tools/kbench.py 8192x8192,4096x4096 480 8 >> gpurun_out/g16_kb.jsonl
done
cat gpurun_out/g16_kb.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bands.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
