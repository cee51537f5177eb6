#!/bin/bash
# stem (K3) floors on the current code: HB_STEM_DBG 1 no stores, 2 no MMA, 4 no TMA (timing only)
for d in 0 1 2 3 4 7 0; do echo "== HB_STEM_DBG=$d"; HB_STEM_DBG=$d timeout 120 python tools/stembench.py 3,64,32,4; HB_STEM_DBG=$d timeout 120 python tools/stembench.py 1,64,64,2; done
timeout 120 python tools/stembench.py 1,1024,32,4
