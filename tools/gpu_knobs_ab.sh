#!/bin/bash
# chain planner knobs on the driver's bench shape (20 flushed ticks), alternated
for r in 1 2 3; do for cfg in "HB_PP_STAGES=4" "HB_PP_STAGES=6" "HB_PP_STAGES=8" "HB_CHAIN_MIN_TILES=1"; do
  env $cfg timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('$cfg', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'], d['parity']['ok'])"
done; done
