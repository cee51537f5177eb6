#!/bin/bash
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x --durations=5 > gpurun_out/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/gputests.log
tail -12 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
