#!/bin/bash
# c5 per rank on one B200: each of the 8 FLOP-balanced member bins at 8192 beds.
mkdir -p gpurun_out
for r in 0 1 2 3 4 5 6 7; do timeout 600 python tools/c5_rank.py $r 8192 2>&1 | tail -1; done | tee gpurun_out/c5.txt
