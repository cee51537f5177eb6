#!/bin/bash
# K4 CTA pairs (tiles paired across beds): throughput A/B, parity, c3 tick A/B
for m in 0 1; do echo "== HB_K4_PAIR=$m"; HB_K4_PAIR=$m timeout 300 python tools/k4wide.py 100 2>&1; done
timeout 900 python -m pytest tests/test_parity_timed_gpu.py -m gpu -x -q -p no:cacheprovider -k "k4_cta_pairs or k4_streamed" 2>&1 | tail -3
for m in 0 1 0 1; do echo "== c3 HB_K4_PAIR=$m"; HB_K4_PAIR=$m timeout 600 python tools/c3prof.py 100 2>&1 | sed -n 1,6p; done
