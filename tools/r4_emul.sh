#!/bin/bash
# Row bands of config 5 on ONE GPU with the quad kernel: the multi-device C-ABI context with
# 1/2/4/8 bands (no kernel waits on another GPU), and bench.py's N-rank path with 2 emulated
# ranks sharing cuda:0 (gloo host barriers).  Band overhead, not a scaling number.
mkdir -p gpurun_out
for n in 1 2 4 8; do
  LIFE_BENCH_DEVICE=0 timeout 600 python bench.py --single-process --gpus $n --steps 2 --warmup 2 > gpurun_out/r4_ctx$n.json 2> gpurun_out/r4_ctx$n.err; echo "ctx $n rc $?"
done
LIFE_BENCH_DEVICE=0 LIFE_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus 2 --steps 2 --warmup 1 > gpurun_out/r4_emul2.json 2> gpurun_out/r4_emul2.err; echo "emul2 rc $?"
python - <<'PY'
import json
for f in ['r4_ctx1','r4_ctx2','r4_ctx4','r4_ctx8','r4_emul2']:
    try:
        j=json.loads(open(f'gpurun_out/{f}.json').read().strip().splitlines()[-1])
        print(f, j['n_gpus'], round(j['value']), j['parity']['ok'], j['config'].get('layout'), j['config'].get('temporal_depth'), round(j['roofline']['frac'],3), round(j['e2e']['value']) if j.get('e2e') else None)
    except Exception as exc:
        print(f, 'ERR', exc)
PY
tail -2 gpurun_out/r4_emul2.err
