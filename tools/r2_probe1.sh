#!/bin/bash
# Round-2 probe: where do config 2 / config 4 packed passes lose against config 5?
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python bench.py --config 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/p1_cfg2.json 2>gpurun_out/p1_cfg2.err
timeout 300 python bench.py --config 4 --steps 2 --warmup 3 --no-cpu --no-e2e > gpurun_out/p1_cfg4.json 2>gpurun_out/p1_cfg4.err
for d in 8 12 16; do
  timeout 300 python tools/kbench.py 16384x16384,40961x12289,65536x65536 480 $d > gpurun_out/p1_kb$d.jsonl
done
for c in 2 4; do
  timeout 600 ncu --set full --clock-control none -k regex:packed_tb -s 12 -c 1 \
    -o /tmp/p1_ncu_cfg$c -f python bench.py --config $c --gens 320 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/p1_ncu_cfg$c.log 2>&1
  ncu -i /tmp/p1_ncu_cfg$c.ncu-rep --page raw --csv > gpurun_out/p1_ncu_cfg${c}_raw.csv
  ncu -i /tmp/p1_ncu_cfg$c.ncu-rep --page details --csv > gpurun_out/p1_ncu_cfg${c}_details.csv
done
ls -la gpurun_out
