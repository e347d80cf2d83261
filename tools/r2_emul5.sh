#!/bin/bash
# Config 5 through bench.py's N>1 path with 2 and 4 ranks emulated on cuda:0 (gloo, host barriers).
mkdir -p gpurun_out
for n in 2 4; do
LIFE_BENCH_DEVICE=0 LIFE_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus $n --steps 2 --warmup 1 > gpurun_out/g15_emul$n.json 2> gpurun_out/g15_emul$n.err
echo "rc $?"
python -c "
import json; j=json.loads(open('gpurun_out/g15_emul$n.json').read().strip().splitlines()[-1])
print(j['n_gpus'], round(j['value']), j['parity']['ok'], j['parity']['kind'], j['roofline']['kernel'], round(j['roofline']['frac'],3), j['e2e']['value'] if j['e2e'] else None)
print([ (r['rank'], r['rows'], round(r['timed_ms']), round(r['interior_ms']), round(r.get('barrier_ms',0)), r.get('pass_sync')) for r in j['ranks']])"
tail -3 gpurun_out/g15_emul$n.err
done
