#!/bin/bash
# K4c chain kernel: parity (HB_CHAIN=1) + A/B on the c2 tick + per-kernel eager profile
mkdir -p gpurun_out
HB_CHAIN=1 timeout 600 python -m pytest tests/test_parity_timed_gpu.py tests/test_engine_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -15
HB_CHAIN=1 timeout 120 python tools/layerprof.py 64 2>&1 | tail -8
HB_CHAIN=1 HB_CHAIN_PROF=1 timeout 120 python tools/chainprof.py 64 > gpurun_out/chainprof.txt 2>&1; tail -3 gpurun_out/chainprof.txt
bash tools/gpu_ab.sh "HB_CHAIN=0" "HB_CHAIN=1"
