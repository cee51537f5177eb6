#!/bin/bash
# ncu evidence for the conv kernels of one c2 tick: per-launch time + DRAM bytes, and a full capture of
# the largest K4b launch (w32 group, block 0 conv2 with identity shortcut, L=7500, 192 rows).
mkdir -p gpurun_out
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:conv_ --csv --log-file gpurun_out/conv_traffic.csv python tools/prof1.py 10,13,30,50 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_pp -s 1 -c 1 \
  -o gpurun_out/prof_pp -f python tools/prof1.py 10,13,30,50 > gpurun_out/ncu_pp.log 2>&1
tail -3 gpurun_out/ncu_pp.log
