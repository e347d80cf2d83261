#!/bin/bash
# Which layout wins where: plain K=16 vs pair K=10 vs quad K=6/5 over torus shapes (kbench wall clock).
mkdir -p gpurun_out
: > gpurun_out/r4s.jsonl
S=16384x65536,16384x262144,32768x32768,32768x16384,65536x16384,131072x8192,24576x24576,49152x49152,8192x131072,32768x65536
KB_PAIR=0 KB_QUAD=0 timeout 300 python tools/kbench.py $S 96 16 >> gpurun_out/r4s.jsonl
KB_PAIR=10 KB_QUAD=0 timeout 300 python tools/kbench.py $S 100 0 >> gpurun_out/r4s.jsonl
KB_QUAD=6 timeout 300 python tools/kbench.py $S 96 0 >> gpurun_out/r4s.jsonl
KB_QUAD=5 timeout 300 python tools/kbench.py $S 100 0 >> gpurun_out/r4s.jsonl
python - <<'PY'
import json, collections
t = collections.defaultdict(dict)
for l in open('gpurun_out/r4s.jsonl'):
    j = json.loads(l)
    key = 'plain16' if j['depth'] == 16 else ('quad' + j['quad'] if j['quad'] not in (None, '0') else 'pair10')
    t[(j['w'], j['h'])][key] = j['gcups']
for k, v in t.items():
    print(k, v)
PY
