#!/bin/bash
# Round-2 first GPU pass: full -m gpu suite (incl. multi-device contexts), smoke, short cfg5 bench.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/g1_smi.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/g1_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/g1_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/g1_smoke.log 2>&1; echo "smoke rc $?" >> gpurun_out/g1_smoke.log
timeout 600 python bench.py --steps 3 --warmup 3 > gpurun_out/g1_bench.json 2> gpurun_out/g1_bench.err; echo "bench rc $?" >> gpurun_out/g1_bench.err
tail -3 gpurun_out/g1_pytest.log; cat gpurun_out/g1_smoke.log gpurun_out/g1_bench.json
