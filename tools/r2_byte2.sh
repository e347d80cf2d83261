#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multi.py -m gpu -x -q -p no:cacheprovider -k "byte or BYTE or small or cfg2 or fuzz or transparen or depth" > gpurun_out/g9_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g9_pytest.log
tail -3 gpurun_out/g9_pytest.log
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
: > gpurun_out/g9_kb.jsonl
for t in 0 1; do
 for d in 4 6 8; do
  LIFE_BYTE_TB2=$t timeout 120 python tools/kbench.py 16384x16384,4096x4096,32768x16384 96 $d 1 | sed "s/^{/{\"tb2\": $t, /" >> gpurun_out/g9_kb.jsonl
 done
done
cat gpurun_out/g9_kb.jsonl
