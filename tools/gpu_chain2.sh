#!/bin/bash
mkdir -p gpurun_out
HB_CHAIN=1 timeout 600 python -m pytest tests/test_parity_timed_gpu.py tests/test_engine_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
for rep in 1 2; do for v in 0 1; do HB_CHAIN=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('chain=$v', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])"; done; done
for v in 0 1; do HB_CHAIN=$v timeout 300 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('20 steps chain=$v', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])"; done
HB_CHAIN=1 HB_CHAIN_PROF=1 timeout 120 python tools/chainprof.py 64 > gpurun_out/chainprof3.txt 2>&1; tail -1 gpurun_out/chainprof3.txt
HB_CHAIN=1 timeout 120 python tools/layerprof.py 64 2>&1 | tail -6
