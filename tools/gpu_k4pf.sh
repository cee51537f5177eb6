#!/bin/bash
S=128:128:3750:1:1,128:128:7500:1:1,256:256:1875:1:1,256:256:1875:2:2,512:512:938:1:1
for l in k4old k4p12 k4p16; do echo "== $l"; HB_LIB_PATH=$PWD/ablib/$l.so K4W_SHAPES=$S timeout 300 python tools/k4wide.py 100 2>&1; done
for l in k4old k4p12 k4p16 k4old k4p12 k4p16; do echo -n "c3 $l: "; HB_LIB_PATH=$PWD/ablib/$l.so timeout 600 python tools/c3prof.py 100 2>&1 | grep "graph tick"; done
