#!/bin/bash
# K4 role cycles on wide shapes (HB_DEBUG=8)
for s in 512:512:938:1:1 256:256:1875:1:1 1024:1024:118:1:1 1024:1024:30:1:1; do
  HB_DEBUG=8 K4W_SHAPES=$s K4W_ITERS=5 timeout 120 python tools/k4wide.py 100 2>&1 | tail -2
done
