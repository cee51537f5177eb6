#!/bin/bash
for d in 0 128 4 1 5 129 133; do HB_PP_DBG=$d timeout 120 python tools/ppdbg_matrix.py 2>&1 | tail -1 | tr '|' '\n'; done
