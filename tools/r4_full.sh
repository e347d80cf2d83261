#!/bin/bash
# Full check: GPU suite, smoke, default bench, reference arm, config-3 lines (auto = quad; pair; plain).
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r4f_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4f_pytest.log
tail -3 gpurun_out/r4f_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r4f_bench.json 2> gpurun_out/r4f_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/r4f_ref.json 2> gpurun_out/r4f_ref.err; echo "ref rc $?"
run() { name=$1; shift; timeout 900 python bench.py --no-cpu "$@" > gpurun_out/r4f_$name.json 2> gpurun_out/r4f_$name.err; echo "$name rc $?"; }
run cfg3_auto --config 3
run cfg3_pair --config 3 --quad-depth 0
run cfg2_quad5 --config 2 --quad-depth 5
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r4f_*.json')):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
        r = j.get('roofline') or {}
        print(f.split('/')[-1], round(j['value'] / 1e3, 2), 'T/s frac', round(r.get('frac') or 0, 3), r.get('kernel'),
              'e2e', round((j.get('e2e') or {}).get('value', 0) / 1e3, 2), 'parity', (j.get('parity') or {}).get('ok'),
              'clk', (j.get('clocks') or {}).get('sm_mhz'), (j.get('clocks') or {}).get('samples'), j.get('cpu_baseline', {}) and (j['cpu_baseline'] or {}).get('value'))
    except Exception as exc:
        print(f, 'ERR', exc)
PY
