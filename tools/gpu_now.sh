#!/bin/bash
# Current-state breakdowns: chain role cycles + timeline (c2), c3 per-launch profile
mkdir -p gpurun_out
HB_CHAIN_PROF=1 timeout 120 python tools/chainprof.py 64 > gpurun_out/chainprof_final.txt 2>&1; tail -2 gpurun_out/chainprof_final.txt
HB_CHAIN_PROF=1 timeout 120 python tools/chaintrace.py 64 > gpurun_out/chaintrace_final.txt 2>&1; head -30 gpurun_out/chaintrace_final.txt
timeout 600 python tools/c3prof.py 100 > gpurun_out/c3prof.txt 2>&1; cat gpurun_out/c3prof.txt | head -50
