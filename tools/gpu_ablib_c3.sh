#!/bin/bash
# A/B of two library builds on the c3 full-zoo tick (K4 serves the wide layers): ablib/old.so vs ablib/new.so
for rep in 1 2; do
for v in old new; do
  HB_LIB_PATH=$PWD/ablib/$v.so timeout 300 python tools/layerprof.py 100 $(python -c "print(','.join(map(str,range(60))))") | tail -1 | sed "s/^/$v /"
done
done
