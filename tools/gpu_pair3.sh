#!/bin/bash
# K4 CTA pairs default on: full GPU suite, compute-sanitizer on the pair kernel, c5 per rank
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/gputests_pair.log 2>&1; tail -3 gpurun_out/gputests_pair.log
{
for t in memcheck racecheck synccheck; do
  echo "== $t (K4 CTA pairs: w64-d16 + 2x w128-d2 + w128-d4, 2 beds)"
  timeout 900 compute-sanitizer --tool $t --print-limit 10 python tests/_tick_worker.py /tmp/san.npz 2 250 1 3 15,16,17,36 2>&1 | tail -3
done
} > gpurun_out/r02_sanitizer_k4pair.txt 2>&1; cat gpurun_out/r02_sanitizer_k4pair.txt
for r in 0 1 3 6; do timeout 600 python tools/c5_rank.py $r 8192 2>&1 | tail -1; done | tee gpurun_out/c5_pair.txt
