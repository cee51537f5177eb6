#!/bin/bash
for d in 0 7 1; do HB_STEM_DBG=$d timeout 120 python tools/stemtick.py 64; HB_CHAIN=0 HB_STEM_DBG=$d timeout 120 python tools/stemtick.py 64; done
for s in 3,64,32,4 1,64,64,2; do timeout 120 python tools/stembench.py $s; done
