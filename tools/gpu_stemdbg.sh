#!/bin/bash
# stem timing experiments: back-to-back launches on zero data under HB_STEM_DBG / HB_STEM settings
timeout 300 python -m pytest tests/test_conv_pp_gpu.py tests/test_conv_gpu.py -k stem -x -q -p no:cacheprovider 2>&1 | tail -2
for cfg in "HB_STEM=1" "HB_STEM_DBG=7" "HB_STEM=0"; do
  echo "== $cfg"; env $cfg timeout 300 python tools/stembench.py
done
