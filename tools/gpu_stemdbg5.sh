#!/bin/bash
# stem (K3): fixed cost vs per-tile slope (bed count sweep), full and skeleton (HB_STEM_DBG=7: no TMA/MMA/stores)
for d in 0 7 1; do echo "== HB_STEM_DBG=$d"; for p in 1 8 16 32 64 128 256; do HB_STEM_DBG=$d timeout 120 python tools/stembench.py 3,$p,32,4; done; done
