#!/bin/bash
mkdir -p gpurun_out
for rep in 1 2; do for v in old new; do for d in 0 1; do HB_PP_DBG=$d HB_LIB_PATH=$PWD/ablib/$v.so timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v dbg=$d', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])"; done; done; done
HB_CHAIN=1 HB_LIB_PATH=$PWD/ablib/new.so timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('new chain', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])"
