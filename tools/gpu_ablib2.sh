#!/bin/bash
timeout 900 python -m pytest tests/test_conv_pp_gpu.py tests/test_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for v in old new; do echo "== $v"; HB_LIB_PATH=$PWD/ablib/$v.so timeout 300 python tools/ppres_bench.py 2>&1 | grep "res=2\|res=1"; done
bash tools/gpu_ablib.sh
