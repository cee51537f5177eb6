#!/bin/bash
# Patient micro-batch size vs tick time (L2 residency of the member chains).
for P in 64 1024; do
for b in 64 0.5 0.25 0.12 0.06; do
  HB_ACT_BUDGET_GB=$b timeout 300 python bench.py --patients $P --steps 20 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/ch.json 2> gpurun_out/ch.err
  python -c "import json;d=json.load(open('gpurun_out/ch.json'));print('P=$P budget=$b', round(d['value']), 'pw/s', round(d['ms_per_step'],3), 'ms')" || tail -3 gpurun_out/ch.err
done; done
