#!/bin/bash
# Final round-2 evidence at HEAD: full GPU suite + smoke, then tools/gpu_r2_evidence.sh (bench lines, launch list,
# ncu traffic + full capture of the chain, sanitizer)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=10 > gpurun_out/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/gputests.log
tail -3 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -2 gpurun_out/smoke.log
bash tools/gpu_r2_evidence.sh
