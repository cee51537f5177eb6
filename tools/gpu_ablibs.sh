#!/bin/bash
# abtick per library build, alternated: tools/gpu_ablibs.sh lib1 lib2 ... (ablib/<lib>.so), 3 rounds
for r in 1 2 3; do for l in "$@"; do
  echo -n "$l: "; HB_LIB_PATH=$PWD/ablib/$l.so AB_ROUNDS=4 timeout 300 python tools/abtick.py "HB_CHAIN=1" 2>&1 | tail -1
done; done
