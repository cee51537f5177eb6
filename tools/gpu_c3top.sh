#!/bin/bash
timeout 600 python tools/c3prof.py 100 > gpurun_out/c3prof_slots.txt 2>&1; sed -n '/top launches/,$p' gpurun_out/c3prof_slots.txt
timeout 900 python -m pytest tests/test_parity_timed_gpu.py -m gpu -x -q -p no:cacheprovider -k "c3 or k4_streamed" 2>&1 | tail -3
