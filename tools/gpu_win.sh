#!/bin/bash
for P in 64 1024; do for w in 1 2; do
  echo -n "P=$P HB_WIN=$w: "; HB_WIN=$w timeout 300 python tools/layerprof.py $P 2>&1 | grep -E "ingest" | head -1
done; done
timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_ingest_cpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
HB_WIN=2 timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
