#!/bin/bash
# K4b iteration: per-layer parity, shape benchmark K4 vs K4b, c2 tick with K4b on/off.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_conv_pp_gpu.py tests/test_engine_gpu.py -x -q -p no:cacheprovider > gpurun_out/pp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pp_tests.log
tail -4 gpurun_out/pp_tests.log
timeout 300 python tools/convbench.py --pp 64 1024 > gpurun_out/convbench_pp.txt 2>&1
cat gpurun_out/convbench_pp.txt
for pp in 1 0; do
  HB_PP=$pp timeout 300 python bench.py --steps 50 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/bench_pp$pp.json 2> gpurun_out/bench_pp$pp.err
  python -c "import json;d=json.load(open('gpurun_out/bench_pp$pp.json'));print('HB_PP=$pp', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['config']['tick_breakdown_ms_eager'], 'conv TF/s', round(d['roofline']['achieved']))"
done
HB_PP=1 timeout 300 python tools/layerprof.py > gpurun_out/layerprof_pp.txt 2>&1; head -70 gpurun_out/layerprof_pp.txt
