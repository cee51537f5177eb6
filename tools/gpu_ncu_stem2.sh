#!/bin/bash
mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:stem_pp -s 3 -c 1 \
  -o gpurun_out/prof_stem3 -f python tools/stembench.py 3,64,32,4 > gpurun_out/ncu_stem3.log 2>&1
HB_STEM_DBG=7 timeout 600 ncu --set full --clock-control none --import-source on -k regex:stem_pp -s 3 -c 1 \
  -o gpurun_out/prof_stem3_floor -f python tools/stembench.py 3,64,32,4 >> gpurun_out/ncu_stem3.log 2>&1
tail -2 gpurun_out/ncu_stem3.log
