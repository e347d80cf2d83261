#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 --cpu-budget 10 > gpurun_out/g8_cfg1.json 2> gpurun_out/g8_cfg1.err
timeout 600 python bench.py --config 2 --engine byte --steps 5 --warmup 3 --cpu-budget 10 > gpurun_out/g8_byte2.json 2> gpurun_out/g8_byte2.err
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --cpu-budget 10 > gpurun_out/g8_cfg2.json 2> gpurun_out/g8_cfg2.err
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --cpu-budget 10 > gpurun_out/g8_cfg4.json 2> gpurun_out/g8_cfg4.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --cpu-budget 10 > gpurun_out/g8_cfg3.json 2> gpurun_out/g8_cfg3.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/g8_ref.json 2> gpurun_out/g8_ref.err
for f in gpurun_out/g8_*.json; do python -c "
import json,sys; j=json.loads(open('$f').read().strip().splitlines()[-1]); r=j.get('roofline',{})
print('$f', round(j['value'],1), r.get('kernel'), r.get('frac'), j.get('clocks'), (j.get('parity') or {}).get('ok'), (j.get('e2e') or {}).get('value'))"; done
