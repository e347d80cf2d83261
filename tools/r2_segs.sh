#!/bin/bash
# Segment-count model check on multi-wave / near-one-wave tori (LIFE_SEGS forces the count).
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
for s in 0 17 35 36 53; do LIFE_SEGS=$s timeout 120 python tools/kbench.py 65536x65536 160 16 | sed "s/^{/{\"segs\": $s, /"; done
for s in 0 13 22 31 49; do LIFE_SEGS=$s timeout 120 python tools/kbench.py 262144x65536 80 16 | sed "s/^{/{\"segs\": $s, /"; done
