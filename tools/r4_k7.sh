#!/bin/bash
# Quad K = 7 by the auto rule: interleaved-path parity, default bench, config 3, ncu capture.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_pair.py tests/test_gpu_pair_bands.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r4k_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4k_pytest.log
tail -3 gpurun_out/r4k_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r4k_bench.json 2> gpurun_out/r4k_bench.err; echo "bench rc $?"
timeout 900 python bench.py --config 3 --no-cpu > gpurun_out/r4k_cfg3.json 2> gpurun_out/r4k_cfg3.err; echo "cfg3 rc $?"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:packed_il_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_cfg5_quad_k7 -f python tools/kbench.py 262144x262144 14 0 > gpurun_out/ncu_cfg5_quad7.log 2>&1
echo "full capture rc $?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv \
  --log-file gpurun_out/launches_cfg5_r03c.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/launches_r03c.log 2>&1
echo "launch list rc $?"
python tools/summarize_launches.py gpurun_out/launches_cfg5_r03c.csv > gpurun_out/launches_cfg5_r03c.md; head -8 gpurun_out/launches_cfg5_r03c.md
python - <<'PY'
import json
for f in ('r4k_bench', 'r4k_cfg3'):
    j = json.loads(open(f'gpurun_out/{f}.json').read().strip().splitlines()[-1]); r = j['roofline']; e = j['e2e']
    print(f, round(j['value']), r['kernel'], round(r['frac'], 4), j['parity']['ok'], 'e2e', round(e['value']), round(e['value'] / j['value'], 3),
          'sync', round(e['sync_call']['value']), 'one', round(e['sync_call']['one_grid_batch']['value']), j['clocks']['sm_mhz'], j['clocks']['reasons'], j['gpu_launches'])
PY
