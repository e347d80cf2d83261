#!/bin/bash
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_bench_contract.py tests/test_cli.py -m gpu -x -q -p no:cacheprovider > gpurun_out/g7_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g7_pytest.log
tail -3 gpurun_out/g7_pytest.log
timeout 600 python bench.py --config 3 --depth 1 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/g7_cfg3_k1.json 2> gpurun_out/g7_cfg3_k1.err
timeout 600 python bench.py --config 1 --steps 5 --warmup 3 > gpurun_out/g7_cfg1.json 2> gpurun_out/g7_cfg1.err
timeout 600 python bench.py --config 2 --engine byte --steps 5 --warmup 3 --no-cpu > gpurun_out/g7_byte2.json 2> gpurun_out/g7_byte2.err
timeout 600 python bench.py --config 2 --engine byte --byte-depth 1 --steps 5 --warmup 3 --no-cpu --no-e2e > gpurun_out/g7_byte2k1.json 2> gpurun_out/g7_byte2k1.err
for f in gpurun_out/g7_*.json; do python -c "
import json,sys; j=json.loads(open('$f').read().strip().splitlines()[-1]); r=j['roofline']
print('$f', round(j['value']), r.get('kernel'), round(r['frac'],3), j['clocks'], j.get('parity',{}).get('ok'))"; done
