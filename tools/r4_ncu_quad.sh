#!/bin/bash
# Quad kernel (stage group 2): parity of the interleaved paths, default bench, then the ncu
# launch list of the bench command and one full capture of a config-5 packed_il_kernel<6, 4> pass.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_pair_bands.py tests/test_gpu_pair.py -m gpu -x -q -p no:cacheprovider > gpurun_out/r4n_pytest.log 2>&1; echo "pytest rc $?" >> gpurun_out/r4n_pytest.log
tail -3 gpurun_out/r4n_pytest.log
timeout 900 python bench.py > gpurun_out/r4n_bench.json 2> gpurun_out/r4n_bench.err; echo "bench rc $?"
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 2500 --csv \
  --log-file gpurun_out/launches_cfg5_r03b.csv python bench.py --steps 2 --warmup 1 --no-cpu > gpurun_out/launches_r03b.log 2>&1
echo "launch list rc $?"
python tools/summarize_launches.py gpurun_out/launches_cfg5_r03b.csv > gpurun_out/launches_cfg5_r03b.md; cat gpurun_out/launches_cfg5_r03b.md
timeout 900 ncu --set full --import-source on --clock-control none -k regex:packed_il_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_cfg5_quad_k6 -f python tools/kbench.py 262144x262144 12 0 > gpurun_out/ncu_cfg5_quad.log 2>&1
echo "full capture rc $?"
python -c "
import json; j=json.loads(open('gpurun_out/r4n_bench.json').read().strip().splitlines()[-1]); r=j['roofline']
print(round(j['value']), r['kernel'], round(r['frac'],4), j['parity']['ok'], round(j['e2e']['value']), j['clocks'], j['gpu_launches'])"
