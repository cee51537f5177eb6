#!/bin/bash
# per-warp vs per-thread epilogue releases (stem acc_empty; K4b/K4c acc_empty, it_empty): ablib/base.so vs ablib/warp.so
for r in 1 2; do for l in base warp; do echo "== $l"; for s in 3,64,32,4 3,256,32,4; do HB_LIB_PATH=$PWD/ablib/$l.so timeout 120 python tools/stembench.py $s; done; HB_STEM_DBG=7 HB_LIB_PATH=$PWD/ablib/$l.so timeout 120 python tools/stembench.py 3,256,32,4; done; done
bash tools/gpu_ablibs.sh base warp 2>&1 | tail -6
for r in 1 2; do for l in base warp; do echo -n "per-layer $l: "; HB_LIB_PATH=$PWD/ablib/$l.so AB_ROUNDS=4 timeout 300 python tools/abtick.py "HB_CHAIN=0" 2>&1 | tail -1; done; done
HB_LIB_PATH=$PWD/ablib/warp.so timeout 900 python -m pytest tests/test_parity_timed_gpu.py tests/test_chain_fuzz_gpu.py tests/test_conv_pp_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -2
