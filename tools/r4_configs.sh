#!/bin/bash
# Bench lines of configs 1-4 (packed / resident / byte engines) with the current library.
mkdir -p gpurun_out
run() { name=$1; shift; timeout 900 python bench.py --no-cpu "$@" > gpurun_out/r4_$name.json 2> gpurun_out/r4_$name.err; echo "$name rc $?"; }
run cfg1_resident --config 1
run cfg2_packed --config 2
run cfg2_pair10 --config 2 --pair-depth 10
run cfg2_pair8 --config 2 --pair-depth 8
run cfg2_byte --config 2 --engine byte
run cfg3_auto --config 3
run cfg3_k16 --config 3 --depth 16
run cfg3_k8 --config 3 --depth 8
run cfg3_k4 --config 3 --depth 4
run cfg3_k1 --config 3 --depth 1
run cfg4_packed --config 4
run cfg4_byte --config 4 --engine byte
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r4_cfg*.json')):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
        r = j.get('roofline') or {}
        print(f.split('/')[-1], round(j['value'] / 1e3, 2), 'T/s frac', round(r.get('frac') or 0, 3), r.get('kernel'),
              'e2e', round((j.get('e2e') or {}).get('value', 0) / 1e3, 2), 'parity', (j.get('parity') or {}).get('ok'),
              'clk', (j.get('clocks') or {}).get('sm_mhz'), (j.get('clocks') or {}).get('samples'))
    except Exception as exc:
        print(f, 'ERR', exc)
PY
