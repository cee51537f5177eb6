#!/bin/bash
# A/B of env settings on the c2 tick: tools/gpu_ab.sh "HB_PP=1" "HB_PP=2" ...
mkdir -p gpurun_out
for rep in 1 2; do
for cfg in "$@"; do
  env $cfg timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$cfg', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])"
done
done
