#!/bin/bash
# Round-2 (session 5) profiles of the pair kernel: launch list of the default bench command,
# then one full capture of a config-5 packed_pair_kernel<10> pass.
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 1200 --csv \
  --log-file gpurun_out/launches_cfg5_r03.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/launches_r03.log 2>&1
echo "launch list rc $?"
python tools/summarize_launches.py gpurun_out/launches_cfg5_r03.csv > gpurun_out/launches_cfg5_r03.md; cat gpurun_out/launches_cfg5_r03.md
KB_PAIR=10 timeout 900 ncu --set full --import-source on --clock-control none -k regex:packed_pair_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_cfg5_pair_k10 -f python tools/kbench.py 262144x262144 20 0 > gpurun_out/ncu_cfg5_pair.log 2>&1
echo "full capture rc $?"
ls -la gpurun_out | head -20
