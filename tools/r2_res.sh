#!/bin/bash
# Temporal-blocked cluster-resident kernel: parity first (short timeouts), then timing.
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_resident.py -x -q -p no:cacheprovider > gpurun_out/g14_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g14_pytest.log
tail -4 gpurun_out/g14_pytest.log
grep -q "rc 0" gpurun_out/g14_pytest.log || exit 1
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
: > gpurun_out/g14_kb.jsonl
for t in 0 1 0 1; do
  LIFE_RESIDENT_TB=$t timeout 120 python tools/kbench.py 1024x1024,512x512,2048x1024,4096x512,2048x2048 800 0 2 | sed "s/^{/{\"tb\": $t, /" >> gpurun_out/g14_kb.jsonl
done
cat gpurun_out/g14_kb.jsonl
unset LIFE_GPU_LIB
timeout 300 python bench.py --config 1 --steps 10 --warmup 3 --no-cpu > gpurun_out/g14_cfg1.json 2> gpurun_out/g14_cfg1.err
cut -c1-300 gpurun_out/g14_cfg1.json
