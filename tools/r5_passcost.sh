#!/bin/bash
# Fixed cost of a pass boundary on one-wave tori: W = 16384, tiles of ~238 rows,
# 1 / 2 / 4 waves per pass (LIFE_SEGS forces the segment count; debug-knob build).
mkdir -p gpurun_out
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
: > gpurun_out/r5_passcost.jsonl
for rep in 1 2; do
for cfg in "16384x16384 69" "16384x32768 138" "16384x65536 276" "16384x131072 552" "16384x16384 0" "16384x32768 0" "16384x65536 0"; do
  set -- $cfg
  for pdl in 1 0; do
    LIFE_SEGS=$2 LIFE_PDL=$pdl timeout 120 python tools/kbench.py $1 960 16 | sed "s/^{/{\"segs\": $2, \"pdl\": $pdl, /" >> gpurun_out/r5_passcost.jsonl
  done
done
done
cat gpurun_out/r5_passcost.jsonl
