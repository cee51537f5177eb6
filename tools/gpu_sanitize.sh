#!/bin/bash
# compute-sanitizer over the serving path: memcheck (whole tick incl. stem, ingest, K4b, aggregate,
# pipelined submit/collect), racecheck + synccheck on K4b (identity-shortcut MMAs, fused head).
mkdir -p gpurun_out
{
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider -k "sliding or pipelined" 2>&1 | tail -3
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_conv_pp_gpu.py -x -q -p no:cacheprovider -k "fused_head or (matches_fp32 and native and 32-32-3750-1-1-2-8) or maxpool" 2>&1 | tail -3
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_conv_pp_gpu.py tests/test_conv_gpu.py -x -q -p no:cacheprovider -k stem 2>&1 | tail -3
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python tools/stembench.py 1,4,32,4 2>&1 | tail -3
timeout 600 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_conv_pp_gpu.py -x -q -p no:cacheprovider -k "matches_fp32 and native and 32-32-3750-1-1-2-8" 2>&1 | tail -3
timeout 600 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_conv_pp_gpu.py -x -q -p no:cacheprovider -k "fused_head" 2>&1 | tail -3
} | tee gpurun_out/sanitize.txt
