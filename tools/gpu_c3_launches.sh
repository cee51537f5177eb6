#!/bin/bash
# c3 (60 members, 100 beds): ncu launch list of one eager tick
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -c 600 --csv \
  --log-file gpurun_out/r02_c3_launches.csv python tools/c3prof.py 100 > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02_c3_launches.csv > gpurun_out/r02_c3_launches_summary.txt; cat gpurun_out/r02_c3_launches_summary.txt
