#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "widths_not or cfg4 or byte or BYTE or cfg2 or transparen or small" > gpurun_out/g17_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g17_pytest.log
tail -5 gpurun_out/g17_pytest.log
grep -q "rc 0" gpurun_out/g17_pytest.log || exit 1
timeout 300 python tools/kbench.py 16384x16384,16383x16384,40961x12289,4097x4096 96 8 1
timeout 600 python bench.py --config 4 --engine byte --steps 3 --warmup 3 --no-cpu > gpurun_out/g17_byte4.json 2> gpurun_out/g17_byte4.err
timeout 600 python bench.py --config 2 --engine byte --steps 5 --warmup 3 --no-cpu > gpurun_out/g17_byte2.json 2> gpurun_out/g17_byte2.err
for f in gpurun_out/g17_byte4.json gpurun_out/g17_byte2.json; do python -c "
import json; j=json.loads(open('$f').read().strip().splitlines()[-1]); r=j['roofline']
print('$f', round(j['value']), r['kernel'], round(r['frac'],3), j['parity'], (j['e2e'] or {}).get('value'))"; done
