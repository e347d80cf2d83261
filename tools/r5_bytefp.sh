#!/bin/bash
# A/B of the byte engine's coarse fill phases (LIFE_BYTE_FILL_PHASES).
mkdir -p gpurun_out
P=$PWD/paper_1209_4408_b200
: > gpurun_out/r5_bytefp.jsonl
for rep in 1 2 3; do
for lib in liblife_gpu.so liblife_gpu_bfp.so; do
  LIFE_GPU_LIB=$P/$lib timeout 300 python tools/kbench.py 16384x16384,40961x12289,32768x16384,8192x8192 96 0 1 >> gpurun_out/r5_bytefp.jsonl
  LIFE_GPU_LIB=$P/$lib timeout 300 python tools/kbench.py 16384x16384,4096x4096 96 4 1 >> gpurun_out/r5_bytefp.jsonl
done
done
python - <<'PY'
import json, collections
d=collections.defaultdict(dict)
for l in open('gpurun_out/r5_bytefp.jsonl'):
    j=json.loads(l); d[(j['w'],j['h'],j['depth'])].setdefault(j['lib'],[]).append(j['gcups'])
for k,v in d.items():
    print(k, {a: round(max(b)/1e3,2) for a,b in v.items()})
PY
LIFE_GPU_LIB=$P/liblife_gpu_bfp.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "byte or BYTE or fuzz or depth or widths" 2>&1 | tail -2
