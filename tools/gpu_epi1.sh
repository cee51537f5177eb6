#!/bin/bash
# new epilogue: parity (K4b unit tests + engine + timed configs, per-layer and chain), then A/B and shape timings
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_conv_pp_gpu.py tests/test_parity_timed_gpu.py tests/test_engine_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
HB_CHAIN=1 timeout 600 python -m pytest tests/test_parity_timed_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
HB_PP_DBG=0 timeout 120 python tools/ppdbg_matrix.py 2>&1 | tail -1 | tr '|' '\n'
bash tools/gpu_ablib.sh
for v in 0 1; do HB_CHAIN=$v timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err; python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('chain=$v', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks'])"; done
HB_CHAIN=1 HB_CHAIN_PROF=1 timeout 120 python tools/chainprof.py 64 > gpurun_out/chainprof2.txt 2>&1; tail -1 gpurun_out/chainprof2.txt
