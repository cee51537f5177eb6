#!/bin/bash
mkdir -p gpurun_out
for cfg in "HB_CHAIN=1" "HB_CHAIN=1 HB_PP_NB=128" "HB_CHAIN=1 HB_PP_NB=160" "HB_CHAIN=1 HB_PP_NB=192" "HB_CHAIN=1 HB_PP_STAGES=3" "HB_CHAIN=1 HB_PP_STAGES=6" "HB_CHAIN=0"; do
  env $cfg timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$cfg', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])"
done
