#!/bin/bash
for lib in liblife_gpu_base.so liblife_gpu.so liblife_gpu_base.so liblife_gpu.so; do
  LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/$lib timeout 600 python bench.py --steps 3 --warmup 2 --no-cpu > gpurun_out/ab.json 2>/dev/null
  python -c "
import json; j=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); e=j['e2e']
print('$lib', round(j['value']), round(e['value']), round(e['sync_call']['one_grid_batch']['value']))"
done
