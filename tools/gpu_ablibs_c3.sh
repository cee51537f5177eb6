#!/bin/bash
# c3 (60-member zoo, 100 beds) tick per library build, alternated
for r in 1 2 3; do for l in "$@"; do
  echo -n "$l: "; HB_LIB_PATH=$PWD/ablib/$l.so AB_SEL=all AB_P=100 AB_ROUNDS=2 AB_TICKS=5 timeout 600 python tools/abtick.py "HB_CHAIN=1" 2>&1 | tail -1
done; done
