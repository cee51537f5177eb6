#!/bin/bash
timeout 300 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 300 python tools/layerprof.py > gpurun_out/layerprof.txt 2>&1; head -3 gpurun_out/layerprof.txt; tail -2 gpurun_out/layerprof.txt
