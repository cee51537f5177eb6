#!/bin/bash
# GPU tests + bench + per-launch profiles with A/B toggles (grouping, PDL)
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
for cfg in "" "HB_NO_PDL=1" "HB_NO_GROUP=1" "HB_NO_GROUP=1 HB_NO_PDL=1"; do
  echo "== $cfg"; env $cfg timeout 300 python tools/layerprof.py 64 | tail -1
done
timeout 600 python bench.py --steps 50 --warmup 5 --no-cpu-baseline > gpurun_out/bench.json 2> gpurun_out/bench.err
python -c "import json; d=json.load(open('gpurun_out/bench.json')); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['config']['tick_latency_ms'])"
timeout 300 python tools/layerprof.py 64 > gpurun_out/layerprof_c2.txt 2>&1
