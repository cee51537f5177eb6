#!/bin/bash
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"elementwise|copy|Copy" --csv python tools/copy_ref.py 2>/dev/null | grep -E "duration|dram__bytes" | awk -F'","' '{gsub(/"/,"",$NF); print $5, $(NF-2), $NF}' | head -40
