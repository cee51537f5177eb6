#!/bin/bash
timeout 600 python -m pytest tests/test_conv_pp_gpu.py tests/test_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -3
bash tools/gpu_ab.sh HB_PP_HEAD=1 HB_PP_HEAD=0
