#!/bin/bash
for v in 1 0; do echo "== HB_PP_RES_PF=$v"; HB_PP_RES_PF=$v timeout 300 python tools/ppres_bench.py 2>&1 | grep -v "pp prof"; done
bash tools/gpu_ab.sh HB_PP_RES_PF=1 HB_PP_RES_PF=0
