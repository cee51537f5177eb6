#!/bin/bash
timeout 600 python -m pytest tests/test_sweep_gpu.py tests/test_runtime_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
HB_SWEEP_RADIX=0 timeout 600 python -m pytest tests/test_sweep_gpu.py -x -q -p no:cacheprovider 2>&1 | tail -1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for r in 1 0; do HB_SWEEP_RADIX=$r timeout 600 python -c "
import bench
r = bench.sweep_bench(0)
print('radix=$r', round(r['n10']['candidates_per_s']), round(r['n16']['candidates_per_s']), r['n10']['best_auc_selector'], r['n10']['best_auc'])
"; done
