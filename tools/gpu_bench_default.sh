#!/bin/bash
# the driver's default bench line (N=1, default K/W) and the reference arm
mkdir -p gpurun_out
timeout 1200 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
python - <<'PY'
import json
d = json.load(open('gpurun_out/bench_default.json'))
print('value', round(d['value']), d['unit'], 'ms', round(d['ms_per_step'], 4), 'steps', d['steps'], 'e2e', round(d['e2e']['value']),
      'roofline', d['roofline']['achieved'], d['roofline']['frac'], 'clocks', d['clocks'])
r = json.load(open('gpurun_out/bench_ref.json')); print('reference', r.get('value'), r.get('unit'))
PY
