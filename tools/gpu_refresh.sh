#!/bin/bash
# c5 per rank (K4 ring slots) + 1024-bed per-layer breakdown
mkdir -p gpurun_out
for r in 0 1 3 6; do timeout 600 python tools/c5_rank.py $r 8192 2>&1 | tail -1; done | tee gpurun_out/c5_slots.txt
HB_CHAIN=0 timeout 300 python tools/layerprof.py 1024 > gpurun_out/layerprof_1024.txt 2>&1; cat gpurun_out/layerprof_1024.txt
