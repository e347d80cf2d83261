#!/bin/bash
# Layout sweep below the auto rule's 2^29-cell threshold with the phased fill.
mkdir -p gpurun_out
: > gpurun_out/r5_rule.jsonl
kb() { tag=$1; shift; timeout 300 python tools/kbench.py "$@" | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/r5_rule.jsonl; }
S=4096x4096,8192x8192,12288x12288,16384x8192,8192x16384,16384x16384,20480x20480,32768x8192,65536x4096,24576x16384,8192x32768,6144x6144
for rep in 1 2; do
  KB_PAIR=0 KB_QUAD=0 kb plain $S 960 16
  KB_PAIR=8 kb pair8 $S 960 0
  KB_PAIR=10 kb pair10 $S 960 0
  KB_PAIR=12 kb pair12 $S 960 0
  KB_QUAD=5 kb quad5 $S 960 0
  KB_QUAD=6 kb quad6 $S 960 0
  KB_QUAD=7 kb quad7 $S 960 0
  kb auto 40961x12289,16383x16383,16384x16384 960 0
  kb k16 65535x65535,131071x65536 320 16
done
python - <<'PY'
import json, collections
d=collections.defaultdict(dict)
for l in open('gpurun_out/r5_rule.jsonl'):
    j=json.loads(l); d[(j['w'],j['h'])].setdefault(j['tag'],[]).append(j['gcups'])
for k,v in d.items():
    print(k, {a: round(max(b)/1e3,2) for a,b in v.items()})
PY
