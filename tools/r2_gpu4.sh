#!/bin/bash
# Full GPU suite + bench lines for configs 2/4/5 and the byte engine.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g4_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g4_pytest.log
tail -3 gpurun_out/g4_pytest.log
for c in 2 4; do timeout 600 python bench.py --config $c --steps 5 --warmup 3 --no-cpu > gpurun_out/g4_bench$c.json 2> gpurun_out/g4_bench$c.err; done
timeout 600 python bench.py --config 2 --engine byte --steps 5 --warmup 3 --no-cpu > gpurun_out/g4_byte2.json 2> gpurun_out/g4_byte2.err
timeout 900 python bench.py --steps 3 --warmup 3 > gpurun_out/g4_bench5.json 2> gpurun_out/g4_bench5.err
cut -c1-400 gpurun_out/g4_*.json
