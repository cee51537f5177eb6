#!/bin/bash
mkdir -p gpurun_out
{
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_parity_timed_gpu.py -x -q -p no:cacheprovider -k "multi_tile_paths_forced and 6" 2>&1 | tail -3
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_parity_timed_gpu.py -x -q -p no:cacheprovider -k "multi_tile_paths_forced and 6" 2>&1 | tail -3
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider -k "sliding or nonfinite" 2>&1 | tail -3
} > gpurun_out/r02_sanitizer_pp.txt 2>&1
cat gpurun_out/r02_sanitizer_pp.txt
