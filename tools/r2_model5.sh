#!/bin/bash
for lib in liblife_gpu_base.so liblife_gpu.so liblife_gpu_base.so liblife_gpu.so; do
  LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/$lib timeout 300 python tools/kbench.py 262144x262144 96 16
done
timeout 900 python bench.py --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/g21_cfg5.json 2>gpurun_out/g21.err
timeout 900 python bench.py --config 3 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/g21_cfg3.json 2>>gpurun_out/g21.err
for f in gpurun_out/g21_cfg5.json gpurun_out/g21_cfg3.json; do python -c "
import json; j=json.loads(open('$f').read().strip().splitlines()[-1]); r=j['roofline']
print('$f', round(j['value']), round(r['frac'],4), round(r['step_frac'],4), j['parity']['ok'])"; done
