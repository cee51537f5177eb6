#!/bin/bash
# Round-2 parity suite at the timed configurations + the touched GPU tests + smoke.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_timed_gpu.py tests/test_engine_gpu.py tests/test_sweep_gpu.py -m gpu -q -p no:cacheprovider --durations=15 > gpurun_out/parity.log 2>&1; echo "rc=$?" >> gpurun_out/parity.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -25 gpurun_out/parity.log; tail -2 gpurun_out/smoke.log
