#!/bin/bash
# sanitizer pass, smoke, the c2 launch list and a full ncu capture of the stem (K3) of the w32 group
mkdir -p gpurun_out
bash tools/gpu_sanitize.sh
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log; tail -2 gpurun_out/smoke.log
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --profile-only --no-cpu-baseline > /dev/null 2>&1
bash tools/gpu_ncu_stem.sh
