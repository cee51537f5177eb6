#!/bin/bash
run() { echo "$*"; env "$@" timeout 120 python tools/convbench.py --pp 192 2>&1 | grep -E "K4b|pp prof" | head -${N:-4}; }
run HB_PP_DBG=16
run HB_PP_DBG=80
