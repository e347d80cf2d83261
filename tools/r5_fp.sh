#!/bin/bash
# A/B of the phase-specialised fill trips (LIFE_FILL_PHASES) on short-tile tori.
mkdir -p gpurun_out
P=$PWD/paper_1209_4408_b200
LIFE_GPU_LIB=$P/liblife_gpu_tl_fp.so timeout 200 python tools/r5_timeline.py 16384 16384 16 8 2>&1 | tail -8
: > gpurun_out/r5_fp.jsonl
for rep in 1 2; do
for lib in liblife_gpu.so liblife_gpu_fp.so; do
  LIFE_GPU_LIB=$P/$lib timeout 200 python tools/kbench.py 16384x16384,8192x8192,4096x4096,24576x24576,32768x16384 960 16 >> gpurun_out/r5_fp.jsonl
  LIFE_GPU_LIB=$P/$lib timeout 200 python tools/kbench.py 16384x16384,8192x8192 960 12 >> gpurun_out/r5_fp.jsonl
done
done
python - <<'PY'
import json
for l in open('gpurun_out/r5_fp.jsonl'):
    j=json.loads(l); print(j['lib'], j['w'], j['h'], j['depth'], j['gcups'])
PY
LIFE_GPU_LIB=$P/liblife_gpu_fp.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "cfg2 or depth or fuzz or small" 2>&1 | tail -2
