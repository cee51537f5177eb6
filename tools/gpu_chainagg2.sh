#!/bin/bash
# fused aggregation with batched partial loads: parity + in-process A/B at 16 / 64 beds
timeout 900 python -m pytest tests/test_parity_timed_gpu.py -m gpu -x -q -p no:cacheprovider -k "fused_aggregation or c2_tick or c2_64 or 1024" 2>&1 | tail -2
for p in 16 64 128; do AB_ROUNDS=6 AB_P=$p timeout 300 python tools/abtick.py "HB_CHAIN_AGG=0" "HB_CHAIN_AGG=1" 2>&1 | tail -2; done
