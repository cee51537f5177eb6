#!/bin/bash
# A/B over (library, env) pairs on the c2 tick: tools/gpu_abx.sh STEPS "lib|ENV=1 ENV2=2" ...  (lib: ablib/<lib>.so, "-" = in-tree)
mkdir -p gpurun_out
steps=$1; shift
for rep in 1 2; do
for spec in "$@"; do
  lib=${spec%%|*}; envs=${spec#*|}
  if [ "$lib" = "-" ]; then L=""; else L="HB_LIB_PATH=$PWD/ablib/$lib.so"; fi
  env $L $envs timeout 300 python bench.py --steps $steps --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
  python -c "import json;d=json.load(open('gpurun_out/ab.json'));print('$spec', round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms', d['clocks']['reasons'])" 2>/dev/null || { echo "$spec FAILED"; tail -3 gpurun_out/ab.err; }
done
done
