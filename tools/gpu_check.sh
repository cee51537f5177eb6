#!/bin/bash
# One GPU round-trip: parity tests, a bench line, the launch list and one full
# ncu capture of the tcgen05 conv kernel.  Run under gpurun from the repo root.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 50 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
    --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --profile-only --no-cpu-baseline > gpurun_out/launches_bench.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 20 -c 3 \
    -o gpurun_out/prof_conv -f python tools/prof1.py 10,13 > gpurun_out/ncu_full.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:window -c 1 \
    -o gpurun_out/prof_window -f python tools/prof1.py 10,13 > gpurun_out/ncu_window.log 2>&1
ls -la gpurun_out
