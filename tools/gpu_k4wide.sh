#!/bin/bash
# K4 wide layers: throughput per shape + one ncu --set full capture (512->512, L=938)
mkdir -p gpurun_out
timeout 300 python tools/k4wide.py 100 2>&1 | tee gpurun_out/k4wide.txt
K4W_SHAPES=512:512:938:1:1 K4W_ITERS=1 timeout 600 ncu --set full --clock-control none -k regex:conv_tc -c 1 \
  -o gpurun_out/k4wide -f python tools/k4wide.py 100 > gpurun_out/k4wide_ncu.log 2>&1; tail -3 gpurun_out/k4wide_ncu.log
