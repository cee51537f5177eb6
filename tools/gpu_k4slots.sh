#!/bin/bash
# K4 streamed-weight slots A/B on the wide shapes + the c3 tick
for n in 2 3 4; do echo "== HB_K4_BSLOTS=$n"; HB_K4_BSLOTS=$n HB_DEBUG=8 timeout 300 python tools/k4wide.py 100 2>&1 | grep -v "^\[prof\]" ; done
for n in 2 4; do echo "== c3 HB_K4_BSLOTS=$n"; HB_K4_BSLOTS=$n timeout 600 python tools/c3prof.py 100 2>&1 | sed -n 1,6p; done
