#!/bin/bash
# Half the warps per SM (tiles twice as tall) on one-wave tori with the phased fill (debug-knob build).
mkdir -p gpurun_out
export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so
: > gpurun_out/r5_warps.jsonl
kb() { tag=$1; shift; timeout 300 python tools/kbench.py "$@" | sed "s/^{/{\"tag\": \"$tag\", /" >> gpurun_out/r5_warps.jsonl; }
S=16384x16384,20480x20480,12288x12288,32768x8192
for rep in 1 2; do
  KB_PAIR=10 kb pair10_w8 $S 960 0
  KB_PAIR=10 LIFE_PAIR_WPB=4 LIFE_PAIR_BPS=1 kb pair10_w4 $S 960 0
  KB_PAIR=10 LIFE_PAIR_WPB=6 LIFE_PAIR_BPS=1 kb pair10_w6 $S 960 0
  KB_PAIR=0 KB_QUAD=0 kb plain16_w8 $S 960 16
  KB_PAIR=0 KB_QUAD=0 LIFE_FAST_WPB=4 LIFE_FAST_BPS=1 kb plain16_w4 $S 960 16
done
python - <<'PY'
import json, collections
d=collections.defaultdict(dict)
for l in open('gpurun_out/r5_warps.jsonl'):
    j=json.loads(l); d[(j['w'],j['h'])].setdefault(j['tag'],[]).append(j['gcups'])
for k,v in d.items():
    print(k, {a: round(max(b)/1e3,2) for a,b in v.items()})
PY
