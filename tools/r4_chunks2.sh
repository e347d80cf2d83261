#!/bin/bash
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pair_bands.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "batch" > gpurun_out/r4c_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4c_pytest.log
tail -4 gpurun_out/r4c_pytest.log
LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_dbg.so LIFE_BATCH_TRACE=1 timeout 600 python tools/r4_trace.py 2>&1 | tail -22
for cfg in 5 3 2; do
  timeout 900 python bench.py --config $cfg --no-cpu > gpurun_out/r4c_cfg$cfg.json 2> gpurun_out/r4c_cfg$cfg.err; echo "cfg $cfg rc $?"
done
python - <<'PY'
import json
for cfg in (5, 3, 2):
    j = json.loads(open(f'gpurun_out/r4c_cfg{cfg}.json').read().strip().splitlines()[-1])
    e = j['e2e']
    print(cfg, round(j['value']), 'e2e', round(e['value']), round(e['value'] / j['value'], 3), 'sync', round(e['sync_call']['value']),
          'one', round(e['sync_call']['one_grid_batch']['value']), round(e['sync_call']['one_grid_batch']['ms_per_call'], 1), j['parity']['ok'])
PY
