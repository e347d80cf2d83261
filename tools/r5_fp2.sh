#!/bin/bash
# A/B of LIFE_FILL_PHASES 0 / 1 / 2 over the engine's kernels (auto rule and forced layouts).
mkdir -p gpurun_out
P=$PWD/paper_1209_4408_b200
: > gpurun_out/r5_fp2.jsonl
kb() { tag=$1; shift; timeout 300 python tools/kbench.py "$@" | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/r5_fp2.jsonl; }
for rep in 1 2; do
for lib in liblife_gpu_fp0.so liblife_gpu.so liblife_gpu_fp2.so; do
  export LIFE_GPU_LIB=$P/$lib
  kb auto 16384x16384,40961x12289,8192x8192,32768x16384,24576x24576 960 0
  kb auto 65536x65536,49152x49152,131072x8192 224 0
  kb auto 262144x262144 56 0
  KB_PAIR=10 kb pair10 16384x16384,32768x16384 960 0
  KB_QUAD=6 kb quad6 16384x16384,32768x16384 960 0
  KB_QUAD=7 kb quad7 16384x16384,32768x16384,32768x32768 960 0
  kb k12 16383x16383,40961x12289 960 12
  kb k16 16383x16383,65535x65535 320 16
done
done
python - <<'PY'
import json, collections
d=collections.defaultdict(dict)
for l in open('gpurun_out/r5_fp2.jsonl'):
    j=json.loads(l); k=(j['tag'],j['w'],j['h'],j['depth']); d[k].setdefault(j['lib'],[]).append(j['gcups'])
for k,v in d.items():
    print(k, {a.replace('liblife_gpu','').replace('.so','') or 'fp1': max(b) for a,b in v.items()})
PY
