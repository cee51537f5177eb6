#!/bin/bash
# full ncu capture of the stem (K3) of the w32 group in one c2 tick (192 rows, 7500 samples, 32 channels)
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:stem_ -c 1 \
  -o gpurun_out/prof_stem -f python tools/prof1.py 10,13,30,50 > gpurun_out/ncu_stem.log 2>&1
tail -3 gpurun_out/ncu_stem.log
