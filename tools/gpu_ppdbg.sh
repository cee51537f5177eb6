#!/bin/bash
timeout 600 python -m pytest tests/test_conv_pp_gpu.py tests/test_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
run() { echo "$*"; env "$@" timeout 120 python tools/convbench.py --pp 192 2>&1 | grep -E "K4b|pp prof" | head -${N:-4}; }
N=16 run HB_PP_DBG=16
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])"
HB_PP_RES_EPI=1 timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('epi-res', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])"
