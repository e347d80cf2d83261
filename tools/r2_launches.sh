#!/bin/bash
# ncu launch list of the default bench command (round 2), and its summary.
mkdir -p gpurun_out
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 800 --csv \
  --log-file gpurun_out/launches_cfg5_r02.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/launches_r02.log 2>&1
echo "rc $?"
python tools/summarize_launches.py gpurun_out/launches_cfg5_r02.csv 2>/dev/null | head -30 || head -5 gpurun_out/launches_cfg5_r02.csv
