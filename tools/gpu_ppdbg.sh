#!/bin/bash
timeout 600 python -m pytest tests/test_conv_pp_gpu.py tests/test_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
HB_PP_CLUSTER=4 timeout 600 python -m pytest tests/test_conv_pp_gpu.py tests/test_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for rep in 1 2; do for cfg in HB_PP_CLUSTER=1 HB_PP_CLUSTER=2 HB_PP_CLUSTER=4; do
env $cfg timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$cfg', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])" || tail -3 gpurun_out/ab.err
done; done
