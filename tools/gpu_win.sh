#!/bin/bash
timeout 600 python -m pytest tests/test_engine_gpu.py tests/test_runtime_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
HB_WIN=1 timeout 600 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
for P in 64 1024; do
  echo -n "P=$P: "; timeout 300 python tools/layerprof.py $P 2>&1 | grep -E "ingest" | head -1
done
