#!/bin/bash
# Phased fill in the long-tile interleaved kernels too (LIFE_FILL_PHASES_IL=2)?
mkdir -p gpurun_out
P=$PWD/paper_1209_4408_b200
: > gpurun_out/r5_il2.jsonl
for rep in 1 2 3; do
for lib in liblife_gpu.so liblife_gpu_il2.so; do
  LIFE_GPU_LIB=$P/$lib timeout 300 python tools/kbench.py 262144x262144 112 0 >> gpurun_out/r5_il2.jsonl
  LIFE_GPU_LIB=$P/$lib timeout 300 python tools/kbench.py 131072x131072,262144x32768,65536x131072 224 0 >> gpurun_out/r5_il2.jsonl
done
done
python - <<'PY'
import json, collections
d=collections.defaultdict(dict)
for l in open('gpurun_out/r5_il2.jsonl'):
    j=json.loads(l); d[(j['w'],j['h'])].setdefault(j['lib'],[]).append(j['gcups'])
for k,v in d.items():
    print(k, {a: [round(x/1e3,2) for x in b] for a,b in v.items()})
PY
