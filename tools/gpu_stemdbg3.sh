#!/bin/bash
# stem floor on the c2 tick: eager per-launch stem time with stores / MMA / TMA removed (garbage outputs)
for d in 0 1 3 7 0; do echo -n "HB_STEM_DBG=$d: "; HB_STEM_DBG=$d timeout 120 python tools/layerprof.py 64 2>&1 | grep -E " stem " | head -2 | tr '\n' ' '; echo; done
