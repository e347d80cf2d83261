#!/bin/bash
# A/B of the specialised drain trips (LIFE_DRAIN_PHASES) in the short-tile interleaved kernels.
mkdir -p gpurun_out
P=$PWD/paper_1209_4408_b200
: > gpurun_out/r5_drain.jsonl
kb() { tag=$1; shift; timeout 300 python tools/kbench.py "$@" | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/r5_drain.jsonl; }
for rep in 1 2 3; do
for lib in liblife_gpu.so liblife_gpu_drain.so; do
  export LIFE_GPU_LIB=$P/$lib
  kb auto 16384x16384,20480x20480,12288x12288,32768x8192,32768x16384,24576x24576 960 0
  KB_QUAD=7 kb quad7 32768x16384 960 0
done
done
python - <<'PY'
import json, collections
d=collections.defaultdict(dict)
for l in open('gpurun_out/r5_drain.jsonl'):
    j=json.loads(l); d[(j['tag'],j['w'],j['h'])].setdefault(j['lib'],[]).append(j['gcups'])
for k,v in d.items():
    print(k, {a: round(max(b)/1e3,2) for a,b in v.items()})
PY
LIFE_GPU_LIB=$P/liblife_gpu_drain.so timeout 900 python -m pytest tests/test_gpu_pair.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
