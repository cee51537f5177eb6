#!/bin/bash
for h in 0 1 0 1; do echo -n "c3 HB_K4_HALF=$h: "; HB_K4_HALF=$h timeout 600 python tools/c3prof.py 100 2>&1 | grep "graph tick"; done
for h in 0 1; do echo -n "c5 rank 0 HB_K4_HALF=$h: "; HB_K4_HALF=$h timeout 600 python tools/c5_rank.py 0 8192 2>&1 | tail -1; done
for r in 3 6; do echo -n "HB_K4_HALF=1: "; timeout 600 python tools/c5_rank.py $r 8192 2>&1 | tail -1; done
