#!/bin/bash
# Full ncu capture (with source-level stall sampling) of one config-2 K=16 pass.
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:packed_tb -s 20 -c 1 \
  -o gpurun_out/ncu_cfg2_k16 -f python tools/kbench.py 16384x16384 160 16 > gpurun_out/ncu_cfg2.log 2>&1
ls -la gpurun_out
