#!/bin/bash
# A/B of two library builds on the c2 tick: ablib/old.so vs ablib/new.so (HB_LIB_PATH), two rounds
mkdir -p gpurun_out
for rep in 1 2 3; do
for v in old new; do
  HB_LIB_PATH=$PWD/ablib/$v.so timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$v', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])"
done
done
