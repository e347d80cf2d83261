#!/bin/bash
mkdir -p gpurun_out
timeout 600 python bench.py --config 2 --engine byte --steps 5 --warmup 3 --no-cpu > gpurun_out/g10_byte2.json 2> gpurun_out/g10_byte2.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:byte_tb2 -s 20 -c 1 \
  -o gpurun_out/ncu_byte2_8 -f python tools/kbench.py 16384x16384 120 8 1 > gpurun_out/ncu_byte2_8.log 2>&1
python -c "
import json; j=json.loads(open('gpurun_out/g10_byte2.json').read().strip().splitlines()[-1]); r=j['roofline']
print(round(j['value']), r['kernel'], r['frac'], r.get('issue_frac'), r.get('vs_one_stream_bound'), j['parity'], j['e2e']['value'], j['e2e']['packed_behind_byte_api']['value'])"
