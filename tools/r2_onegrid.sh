#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/g18_cfg5.json 2> gpurun_out/g18_cfg5.err
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/g18_cfg2.json 2> gpurun_out/g18_cfg2.err
for f in gpurun_out/g18_cfg5.json gpurun_out/g18_cfg2.json; do python -c "
import json; j=json.loads(open('$f').read().strip().splitlines()[-1]); e=j['e2e']
print('$f', round(j['value']), round(e['value']), round(e['sync_call']['value']), round(e['sync_call']['one_grid_batch']['value']), round(e['sync_call']['ms_per_call'],1), round(e['sync_call']['one_grid_batch']['ms_per_call'],1), j['parity']['ok'], j['clocks'])"; done
