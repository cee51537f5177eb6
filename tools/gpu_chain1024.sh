#!/bin/bash
# The chain at 1024 beds with bed-chunked queues (L2-sized chunks) vs per-layer launches
AB_P=1024 AB_ROUNDS=4 AB_TICKS=5 timeout 900 python tools/abtick.py "HB_CHAIN=0" "HB_CHAIN=1 HB_CHAIN_CHUNKS=2" \
  "HB_CHAIN=1 HB_CHAIN_CHUNKS=8" "HB_CHAIN=1 HB_CHAIN_CHUNKS=16" "HB_CHAIN=1 HB_CHAIN_CHUNKS=32" \
  "HB_CHAIN=1 HB_CHAIN_CHUNKS=16 HB_CHAIN_CHUNK_MIN=32" 2>&1 | tail -8
