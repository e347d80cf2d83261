#!/bin/bash
# Final check of the round: GPU suite, smoke, default bench + reference arm, config lines,
# launch list of the bench command and a full ncu capture of config 2's pair kernel.
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r5h_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r5h_pytest.log
tail -3 gpurun_out/r5h_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 600 python bench.py --impl reference > gpurun_out/r5h_ref.json 2> gpurun_out/r5h_ref.err; echo "ref rc $?"
timeout 900 python bench.py > gpurun_out/r5h_bench.json 2> gpurun_out/r5h_bench.err; echo "bench rc $?"
run() { name=$1; shift; timeout 900 python bench.py --no-cpu "$@" > gpurun_out/r5h_$name.json 2> gpurun_out/r5h_$name.err; echo "$name rc $?"; }
run cfg2_auto --config 2
run cfg4_auto --config 4
run cfg2_byte --config 2 --engine byte
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv \
  --log-file gpurun_out/launches_cfg5_r04b.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/launches_r04b.log 2>&1
echo "launch list rc $?"
python tools/summarize_launches.py gpurun_out/launches_cfg5_r04b.csv > gpurun_out/launches_cfg5_r04b.md; head -12 gpurun_out/launches_cfg5_r04b.md
timeout 900 ncu --set full --import-source on --clock-control none -k regex:packed_il_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_cfg5_quad_k7_r04 -f python tools/kbench.py 262144x262144 14 0 > gpurun_out/ncu_cfg5_quad_k7_r04.log 2>&1
echo "full capture rc $?"
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r5h_*.json')):
    try:
        j = json.loads(open(f).read().strip().splitlines()[-1])
        r = j.get('roofline') or {}
        print(f.split('/')[-1], round(j['value'] / 1e3, 2), 'T/s frac', round(r.get('frac') or 0, 3), r.get('kernel'),
              'e2e', round((j.get('e2e') or {}).get('value', 0) / 1e3, 2), 'parity', (j.get('parity') or {}).get('ok'),
              'clk', (j.get('clocks') or {}).get('sm_mhz'), (j.get('clocks') or {}).get('samples'), (j.get('cpu_baseline') or {}).get('value'))
    except Exception as exc:
        print(f, 'ERR', exc)
PY
