#!/bin/bash
# K4c over bed chunks above HB_CHAIN_MAX_P beds: parity, then in-process A/B against the per-layer path
timeout 1200 python -m pytest tests/test_parity_timed_gpu.py -m gpu -x -q -p no:cacheprovider -k "bed_chunks or 1024 or fused_aggregation or c2_64" 2>&1 | tail -3
for p in 192 256 512 1024; do echo "== P=$p"; AB_ROUNDS=4 AB_P=$p timeout 600 python tools/abtick.py "HB_CHAIN=0" "HB_CHAIN_CHUNK_P=64" "HB_CHAIN_CHUNK_P=96" "HB_CHAIN_CHUNK_P=128" "HB_CHAIN=1 HB_CHAIN_CHUNK_P=0" 2>&1 | tail -5; done
