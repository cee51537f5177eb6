#!/bin/bash
timeout 900 compute-sanitizer --tool racecheck --print-limit 200 python tests/_tick_worker.py /tmp/san.npz 2 250 1 3 15,16,17,36 2>&1 | grep -E "access at|SUMMARY" | sed 's/\[[0-9]* hazards\]//' | sort | uniq -c
for s in 512:512:938:1:1 128:128:3750:1:1 1024:1024:59:1:1; do HB_DEBUG=8 K4W_SHAPES=$s K4W_ITERS=5 timeout 120 python tools/k4wide.py 100 2>&1 | tail -2; done
K4W_SHAPES=128:128:3750:1:1 K4W_ITERS=1 timeout 600 ncu --set full --clock-control none -k regex:conv_tc -c 1 -o gpurun_out/k4pair128 -f python tools/k4wide.py 100 > /dev/null 2>&1
K4W_SHAPES=512:512:938:1:1 K4W_ITERS=1 timeout 600 ncu --set full --clock-control none -k regex:conv_tc -c 1 -o gpurun_out/k4pair512 -f python tools/k4wide.py 100 > /dev/null 2>&1
ls gpurun_out/
