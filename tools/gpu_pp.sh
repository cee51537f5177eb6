#!/bin/bash
# K4b iteration: per-layer parity, shape benchmark K4 vs K4b, c2 tick.
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_conv_pp_gpu.py tests/test_engine_gpu.py -x -q -p no:cacheprovider > gpurun_out/pp_tests.log 2>&1; echo "rc=$?" >> gpurun_out/pp_tests.log
tail -4 gpurun_out/pp_tests.log
timeout 300 python tools/convbench.py --pp ${PP_SIZES:-64 192} > gpurun_out/convbench_pp.txt 2>&1
grep K4b gpurun_out/convbench_pp.txt
for cfg in ${AB:-HB_PP=1}; do
  env $cfg timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$cfg', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])"
done
