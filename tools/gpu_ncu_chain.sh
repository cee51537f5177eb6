#!/bin/bash
# ncu full capture of the K4c chain launch (c2 tick, 64 beds)
mkdir -p gpurun_out
HB_CHAIN=1 timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_pp -c 1 \
  -o gpurun_out/prof_chain -f python tools/prof1.py 10,13,30,50 > gpurun_out/ncu_chain.log 2>&1
tail -3 gpurun_out/ncu_chain.log
python tools/ncu_summary.py gpurun_out/prof_chain.ncu-rep > gpurun_out/ncu_chain_summary.txt 2>&1
head -40 gpurun_out/ncu_chain_summary.txt
