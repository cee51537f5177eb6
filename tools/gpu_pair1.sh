#!/bin/bash
# K4 CTA pairs: smoke on one wide shape, then throughput A/B and parity
HB_K4_PAIR=1 K4W_SHAPES=512:512:938:1:1 K4W_ITERS=3 timeout 120 python tools/k4wide.py 100 2>&1 | tail -3
echo "rc=$?"
for m in 0 1; do echo "== HB_K4_PAIR=$m"; HB_K4_PAIR=$m timeout 300 python tools/k4wide.py 100 2>&1; done
timeout 900 python -m pytest tests/test_parity_timed_gpu.py -m gpu -x -q -p no:cacheprovider -k "k4_cta_pairs or k4_streamed" 2>&1 | tail -5
