#!/bin/bash
# stem (K3) parity under both kernels, the engine tests, the c2 tick A/B and the eager per-layer profile
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_conv_pp_gpu.py tests/test_conv_gpu.py -k stem -x -q -p no:cacheprovider 2>&1 | tail -2
HB_STEM=0 timeout 300 python -m pytest tests/test_conv_pp_gpu.py tests/test_conv_gpu.py -k stem -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -2
timeout 120 python tools/stembench.py
bash tools/gpu_ab.sh HB_STEM=1 HB_STEM=0
timeout 300 python tools/layerprof.py > gpurun_out/layerprof.txt 2>&1; head -3 gpurun_out/layerprof.txt; sed -n 19,20p gpurun_out/layerprof.txt; tail -1 gpurun_out/layerprof.txt
