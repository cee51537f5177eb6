#!/bin/bash
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_runtime_gpu.py -m gpu -q -p no:cacheprovider -k wallclock 2>&1 | tail -2
bash tools/gpu_ablib.sh
HB_LIB_PATH=$PWD/ablib/old.so timeout 300 python tools/layerprof.py 64 > gpurun_out/layerprof_old.txt 2>&1
HB_LIB_PATH=$PWD/ablib/new.so timeout 300 python tools/layerprof.py 64 > gpurun_out/layerprof_new.txt 2>&1
tail -1 gpurun_out/layerprof_old.txt gpurun_out/layerprof_new.txt
