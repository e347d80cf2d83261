#!/bin/bash
mkdir -p gpurun_out
: > gpurun_out/g13_kb.jsonl
for lib in liblife_gpu.so liblife_gpu_ufma.so liblife_gpu.so liblife_gpu_ufma.so; do
  LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/$lib timeout 120 python tools/kbench.py 16384x16384,32768x16384 96 8 1 >> gpurun_out/g13_kb.jsonl
done
cat gpurun_out/g13_kb.jsonl
LIFE_GPU_LIB=$PWD/paper_1209_4408_b200/liblife_gpu_ufma.so timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "byte or BYTE or cfg2 or transparen" 2>&1 | tail -2
# multi-device C-ABI context, bands emulated on cuda:0: decomposition overhead
for n in 1 2 4 8; do
  LIFE_BENCH_DEVICE=0 timeout 600 python bench.py --single-process --gpus $n --steps 2 --warmup 2 > gpurun_out/g13_ctx$n.json 2> gpurun_out/g13_ctx$n.err
done
for n in 1 2 4 8; do python -c "
import json; j=json.loads(open('gpurun_out/g13_ctx$n.json').read().strip().splitlines()[-1])
print($n, round(j['value']), j['parity']['ok'], [round(b['run_ms'],1) for b in j['bands']], [round(b['interior_ms'],1) for b in j['bands']], [round(b['edge_ms'],2) for b in j['bands']])"; done
