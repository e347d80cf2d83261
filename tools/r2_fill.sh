#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/g11_kb.jsonl
for lib in liblife_gpu.so liblife_gpu_fill.so liblife_gpu.so liblife_gpu_fill.so; do
  LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/$lib timeout 120 python tools/kbench.py 16384x16384,4096x4096,32768x16384 96 8 1 >> gpurun_out/g11_kb.jsonl
  LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/$lib timeout 120 python tools/kbench.py 16384x16384,4096x4096 96 4 1 >> gpurun_out/g11_kb.jsonl
done
cat gpurun_out/g11_kb.jsonl
LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_fill.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "byte or BYTE or small or cfg2 or fuzz or transparen or depth" 2>&1 | tail -2
