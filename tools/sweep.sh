#!/bin/bash
# Kernel-variant / depth sweep on one GPU (used under gpurun); one JSON line per run.
# usage: tools/sweep.sh CONFIG GENS "LIBS" "DEPTHS"
cfg=${1:-3}; gens=${2:-256}; libs=${3:-default}; depths=${4:-"4 8 12 16"}
out=gpurun_out/sweep.jsonl
for lib in $libs; do
  for d in $depths; do
    if [ "$lib" = default ]; then unset LIFE_GPU_LIB; else export LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_$lib.so; fi
    line=$(timeout 300 python bench.py --config $cfg --gens $gens --depth $d --steps 3 --warmup 1 --no-e2e --no-cpu 2>gpurun_out/sweep_err.log | tail -1)
    python - "$lib" "$d" "$line" >> $out <<'PY'
import json, sys
lib, d, line = sys.argv[1], sys.argv[2], sys.argv[3]
try:
    j = json.loads(line)
    print(json.dumps({"lib": lib, "depth": int(d), "gcups": round(j["value"], 1),
                      "frac": round(j["roofline"]["frac"], 4), "kern_ms": j["roofline"]["mean_launch_ms"],
                      "peak": j["roofline"]["peak"], "clocks": j["clocks"]}))
except Exception as e:
    print(json.dumps({"lib": lib, "depth": int(d), "error": repr(e), "line": line[:300]}))
PY
  done
done
cat $out
