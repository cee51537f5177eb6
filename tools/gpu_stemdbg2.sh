#!/bin/bash
for cfg in "HB_STEM_DBG=1" "HB_STEM_DBG=2" "HB_STEM_DBG=4" "HB_STEM_DBG=3" "HB_STEM_DBG=5" "HB_STEM_DBG=6"; do
  echo "== $cfg"; env $cfg timeout 120 python tools/stembench.py 2>&1 | head -2
done
timeout 300 python -m pytest tests/test_conv_pp_gpu.py -k stem -x -q -p no:cacheprovider 2>&1 | grep -i "error\|assert" | head -5
