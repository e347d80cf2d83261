#!/bin/bash
# Full ncu capture (source-level stall sampling) of one config-2 byte_tb_kernel<6> pass.
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on --clock-control none -k regex:byte_tb -s 20 -c 1 \
  -o gpurun_out/ncu_byte6 -f python tools/kbench.py 16384x16384 120 6 1 > gpurun_out/ncu_byte6.log 2>&1
ls -la gpurun_out/ncu_byte6*
