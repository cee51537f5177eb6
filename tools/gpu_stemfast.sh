#!/bin/bash
timeout 600 python -m pytest tests/test_conv_pp_gpu.py tests/test_conv_gpu.py -m gpu -x -q -p no:cacheprovider -k stem 2>&1 | tail -2
timeout 600 python -m pytest tests/test_parity_timed_gpu.py -m gpu -x -q -p no:cacheprovider -k "c2_64 or c1_one" 2>&1 | tail -2
for r in 1 2; do for l in stemold stemnew; do echo -n "$l: "; HB_LIB_PATH=$PWD/ablib/$l.so timeout 120 python tools/layerprof.py 64 2>&1 | grep -E " stem |graph tick" | tr '\n' ' '; echo; done; done
bash tools/gpu_ablibs.sh stemold stemnew 2>&1 | tail -6
