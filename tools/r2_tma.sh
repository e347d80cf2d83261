#!/bin/bash
mkdir -p gpurun_out
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
: > gpurun_out/g6_kb.jsonl
for t in 0 1; do
  LIFE_STEP1_TMA=$t timeout 60 python tools/kbench.py 65536x65536,16384x16384,262144x16384 64 1 | sed "s/^{/{\"tma\": $t, /" >> gpurun_out/g6_kb.jsonl
done
cat gpurun_out/g6_kb.jsonl
LIFE_STEP1_TMA=1 timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "depth or vector or known" 2>&1 | tail -3
