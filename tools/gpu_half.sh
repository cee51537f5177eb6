#!/bin/bash
# K4 half pairs (M = 128 over the pair, 64 rows per CTA) on the deep layers
S=1024:1024:59:1:1,1024:1024:30:1:1,1024:1024:118:2:2,1024:1024:59:2:0,512:512:59:1:1,1024:1024:118:1:1
HB_K4_HALF=1 K4W_SHAPES=1024:1024:59:1:1 K4W_ITERS=3 timeout 120 python tools/k4wide.py 100 2>&1 | tail -2; echo "rc=$?"
for h in 0 1; do echo "== HB_K4_HALF=$h"; HB_K4_HALF=$h K4W_SHAPES=$S timeout 300 python tools/k4wide.py 100 2>&1; done
timeout 900 python -m pytest tests/test_parity_timed_gpu.py -m gpu -x -q -p no:cacheprovider -k "k4_cta or k4_streamed or lane_caps" 2>&1 | tail -3
