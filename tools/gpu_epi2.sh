#!/bin/bash
mkdir -p gpurun_out
for v in old new; do HB_LIB_PATH=$PWD/ablib/$v.so timeout 300 python tools/layerprof.py 64 > gpurun_out/layerprof_$v.txt 2>&1; done
paste gpurun_out/layerprof_old.txt gpurun_out/layerprof_new.txt | awk -F'\t' '{printf "%-60s | %s\n", substr($1,1,40), substr($2,16,40)}'
for v in old new; do for d in 0 1; do HB_PP_DBG=$d HB_LIB_PATH=$PWD/ablib/$v.so timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v dbg=$d', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks'])"; done; done
