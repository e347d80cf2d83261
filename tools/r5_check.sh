#!/bin/bash
# Phased fill + pair layout from 2^27 cells: GPU suite, smoke, bench lines of configs 2 / 4 / 1 / 3, split-launch shapes.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r5_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r5_pytest.log
tail -3 gpurun_out/r5_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
run() { name=$1; shift; timeout 900 python bench.py --no-cpu "$@" > gpurun_out/r5_$name.json 2> gpurun_out/r5_$name.err; echo "$name rc $?"; }
run cfg2_auto --config 2
run cfg2_plain --config 2 --pair-depth 0 --quad-depth 0
run cfg4_auto --config 4
run cfg3_auto --config 3
run cfg1_auto --config 1
timeout 300 python tools/kbench.py 65535x65535,131071x65536,16383x16383,40961x12289 320 0
timeout 300 python tools/kbench.py 65535x65535,131071x65536,16383x16383 320 16
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r5_cfg*.json')):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
        r = j.get('roofline') or {}
        print(f.split('/')[-1], round(j['value'] / 1e3, 2), 'T/s frac', round(r.get('frac') or 0, 3), r.get('kernel'),
              'e2e', round((j.get('e2e') or {}).get('value', 0) / 1e3, 2), 'parity', (j.get('parity') or {}).get('ok'),
              'clk', (j.get('clocks') or {}).get('sm_mhz'), (j.get('clocks') or {}).get('samples'))
    except Exception as exc:
        print(f, 'ERR', exc)
PY
