#!/bin/bash
# TMA step1 kernel: parity + A/B timing; config-3 depth table bench lines.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_bands.py -m gpu -x -q -p no:cacheprovider -k "depth or vector or cfg3 or local_bands or packed_run or known" > gpurun_out/g5_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g5_pytest.log
tail -3 gpurun_out/g5_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" >> gpurun_out/g5_pytest.log 2>&1
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
: > gpurun_out/g5_kb.jsonl
for t in 0 1 0 1; do
  LIFE_STEP1_TMA=$t timeout 300 python tools/kbench.py 65536x65536,16384x16384,262144x16384 64 1 | sed "s/^{/{\"tma\": $t, /" >> gpurun_out/g5_kb.jsonl
done
cat gpurun_out/g5_kb.jsonl
unset LIFE_GPU_LIB
for d in 1 4 8 16; do
  timeout 600 python bench.py --config 3 --depth $d --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/g5_cfg3_k$d.json 2> gpurun_out/g5_cfg3_k$d.err
done
cut -c1-250 gpurun_out/g5_cfg3_k*.json
