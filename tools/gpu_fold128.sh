#!/bin/bash
S=128:128:3750:1:1,128:128:3750:1:0,128:128:938:1:1,128:128:7500:1:1,128:128:1875:2:2
for f in 0 1; do echo "== HB_FOLD128=$f"; HB_FOLD128=$f K4W_SHAPES=$S timeout 300 python tools/k4wide.py 100 2>&1; done
for f in 0 1 0 1; do echo "== c3 HB_FOLD128=$f"; HB_FOLD128=$f timeout 600 python tools/c3prof.py 100 2>&1 | sed -n 1,6p; done
