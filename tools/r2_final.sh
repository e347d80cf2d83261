#!/bin/bash
# Round-2 final check: full GPU suite, smoke, default bench line, reference arm.
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/final_pytest.log
tail -3 gpurun_out/final_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 1200 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc $?"
timeout 600 python bench.py --impl reference > gpurun_out/final_ref.json 2> gpurun_out/final_ref.err; echo "ref rc $?"
python -c "
import json; j=json.loads(open('gpurun_out/final_bench.json').read().strip().splitlines()[-1]); r=j['roofline']
print(round(j['value']), round(r['frac'],4), j['parity']['ok'], round(j['e2e']['value']), j['cpu_baseline']['value'], j['clocks'], j['gpu_launches'])
k=json.loads(open('gpurun_out/final_ref.json').read().strip().splitlines()[-1]); print('ref', k['value'], k['cpu_baseline']['sample'])"
