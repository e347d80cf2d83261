#!/bin/bash
# bench.py's N-rank path with 2 / 4 ranks sharing cuda:0 (gloo for the collectives of the
# harness): default pass sync (host barriers under gloo) vs the stream-memory-operation flags
# each rank bumps in its neighbours' IPC buffers.  Time-sliced ranks: parity and the
# machinery's cost, not a scaling number.
mkdir -p gpurun_out
for n in 2 4; do
for sync in neighbour flag_overlap; do
  LIFE_BENCH_DEVICE=0 LIFE_BENCH_BACKEND=gloo timeout 900 python bench.py --gpus $n --steps 2 --warmup 1 --no-e2e --pass-sync $sync > gpurun_out/r5_emul${n}_$sync.json 2> gpurun_out/r5_emul${n}_$sync.err; echo "emul $n $sync rc $?"
done
done
python - <<'PY'
import json, glob
for f in sorted(glob.glob('gpurun_out/r5_emul*_*.json')):
    try:
        j=json.loads(open(f).read().strip().splitlines()[-1])
        print(f.split('/')[-1], j['n_gpus'], round(j['value']), j['parity']['ok'], j['config'].get('layout'), [r.get('pass_sync') for r in j.get('ranks', [])][:1])
    except Exception as exc:
        print(f, 'ERR', exc)
PY
