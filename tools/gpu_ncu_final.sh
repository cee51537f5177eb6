#!/bin/bash
# ncu on the final chain kernel (aggregation fused): DRAM traffic per tick + full capture summary
mkdir -p gpurun_out
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"conv_|chain_" --csv --log-file gpurun_out/conv_traffic.csv python tools/prof1.py 10,13,30,50 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/conv_traffic.csv gpurun_out/ncu_conv_summary.json | head -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_pp -c 1 \
  -o gpurun_out/prof_chain -f python tools/prof1.py 10,13,30,50 > gpurun_out/ncu_chain.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_chain.ncu-rep > gpurun_out/r02_ncu_chain_summary.txt 2>&1
head -12 gpurun_out/r02_ncu_chain_summary.txt
