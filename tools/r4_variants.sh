#!/bin/bash
# Quad-kernel variants (stage group size, prefetch depth) against the base build, kbench wall clock.
mkdir -p gpurun_out
: > gpurun_out/r4v.jsonl
for rep in 1 2; do
for v in base qg2 qg3 pf4 pf8; do
  export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_v_$v.so
  for d in 5 6; do
    KB_QUAD=$d timeout 200 python tools/kbench.py 262144x262144,65536x65536 $((d*20)) 0 >> gpurun_out/r4v.jsonl
  done
done
done
python - <<'PY'
import json, collections
best = collections.defaultdict(float)
for l in open('gpurun_out/r4v.jsonl'):
    j = json.loads(l)
    k = (j['lib'], j['quad'], j['w'])
    best[k] = max(best[k], j['gcups'])
for k in sorted(best):
    print(k, best[k])
PY
