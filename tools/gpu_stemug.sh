#!/bin/bash
# stem epilogue: units per TMEM load set (HB_STEM_UG 1 = x8 x two sets, 4 = x32 x one set)
for r in 1 2; do for u in 1 4; do echo "== HB_STEM_UG=$u"; for s in 3,64,32,4 1,64,64,2 3,256,32,4 1,1024,32,4; do HB_STEM_UG=$u timeout 120 python tools/stembench.py $s; done; HB_STEM_DBG=7 HB_STEM_UG=$u timeout 120 python tools/stembench.py 3,256,32,4; done; done
AB_ROUNDS=6 timeout 300 python tools/abtick.py "HB_STEM_UG=1" "HB_STEM_UG=4" 2>&1 | tail -3
HB_STEM_UG=4 timeout 900 python -m pytest tests/test_conv_pp_gpu.py tests/test_conv_gpu.py tests/test_engine_gpu.py -m gpu -x -q -p no:cacheprovider -k "stem or sliding or c3" 2>&1 | tail -2
HB_STEM_UG=4 timeout 900 python -m pytest tests/test_parity_timed_gpu.py -m gpu -x -q -p no:cacheprovider -k "c2_64 or c1 or 1024" 2>&1 | tail -2
