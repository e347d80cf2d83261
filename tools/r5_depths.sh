#!/bin/bash
# Depth sweeps with the phased fill: all-paths kernel on config 4 / 16383^2, pair depth on config-2-class tori.
mkdir -p gpurun_out
: > gpurun_out/r5_depths.jsonl
kb() { tag=$1; shift; timeout 300 python tools/kbench.py "$@" | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/r5_depths.jsonl; }
for rep in 1 2; do
  for d in 8 10 12 14 16; do kb plain$d 40961x12289,16383x16383 960 $d; done
  for d in 9 10 11 12; do KB_PAIR=$d kb pair$d 16384x16384,20480x20480,32768x16384,12288x12288 960 0; done
done
python - <<'PY'
import json, collections
d=collections.defaultdict(dict)
for l in open('gpurun_out/r5_depths.jsonl'):
    j=json.loads(l); d[(j['w'],j['h'])].setdefault(j['tag'],[]).append(j['gcups'])
for k,v in d.items():
    print(k, {a: round(max(b)/1e3,2) for a,b in v.items()})
PY
