#!/bin/bash
timeout 600 python -m pytest tests/test_conv_pp_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
run() { echo "$*"; env "$@" timeout 120 python tools/convbench.py --pp 192 2>&1 | grep -E "K4b|pp prof" | head -${N:-4}; }
run HB_PP_DBG=16
run HB_PP_DBG=24
run HB_PP_DBG=48
