#!/bin/bash
mkdir -p gpurun_out
timeout 300 python tools/chaintrace.py 64 > gpurun_out/chaintrace.txt 2>&1; cat gpurun_out/chaintrace.txt | tail -28
HB_CHAIN_OPTS=3 timeout 300 python tools/chaintrace.py 64 2>&1 | head -1
bash tools/gpu_abx.sh 100 "-|HB_CHAIN_OPTS=0" "-|HB_CHAIN_OPTS=1" "-|HB_CHAIN_OPTS=2" "-|HB_CHAIN_OPTS=3"
