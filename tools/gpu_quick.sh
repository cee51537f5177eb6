#!/bin/bash
# Full GPU suite + one bench line (with side measurements) + eager per-layer profile.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gpu_all.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_all.log
tail -3 gpurun_out/gpu_all.log
timeout 600 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
python - <<'PY'
import json
d = json.load(open('gpurun_out/bench.json'))
c = d['config']
print('c2', round(d['value']), 'pw/s', round(d['ms_per_step'], 4), 'ms; e2e', round(d['e2e']['value']), 'conv TF/s', round(d['roofline']['achieved']), 'frac', round(d['roofline']['frac'], 3))
print('1024 beds', c.get('beds_1024')); print('c3', c.get('c3_full_zoo_100_beds')); print('clocks', d['clocks'])
PY
timeout 300 python tools/layerprof.py > gpurun_out/layerprof.txt 2>&1; tail -1 gpurun_out/layerprof.txt
