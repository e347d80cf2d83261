#!/bin/bash
# Round-2: bench multi-rank contract, parity in the line, split-launch goldens.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_bench_contract.py tests/test_gpu_parity.py -m gpu -x -q -p no:cacheprovider -k "bench or split or cfg2 or cfg4 or gpus or single or parity_line or one_gpu" > gpurun_out/g2_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g2_pytest.log
timeout 600 python bench.py --steps 3 --warmup 3 --no-cpu > gpurun_out/g2_bench5.json 2> gpurun_out/g2_bench5.err
timeout 600 python bench.py --config 2 --steps 5 --warmup 3 --no-cpu > gpurun_out/g2_bench2.json 2> gpurun_out/g2_bench2.err
timeout 600 python bench.py --config 4 --steps 3 --warmup 3 --no-cpu > gpurun_out/g2_bench4.json 2> gpurun_out/g2_bench4.err
tail -5 gpurun_out/g2_pytest.log; cat gpurun_out/g2_bench*.json | cut -c1-600
