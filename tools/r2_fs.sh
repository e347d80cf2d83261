#!/bin/bash
mkdir -p gpurun_out
LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_fs.so timeout 300 python tools/kbench.py 16384x16384,16383x16384 96 8 1
timeout 300 python tools/kbench.py 16384x16384,16383x16384 96 8 1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:byte_tb2 -s 5 -c 1 -o gpurun_out/ncu_byteseam -f python tools/kbench.py 16383x16384 40 8 1 > /dev/null 2>&1
ls -la gpurun_out/ncu_byteseam*
