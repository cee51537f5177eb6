#!/bin/bash
# chain queue bed chunks (HB_CHAIN_CHUNKS) 2 vs 3 vs 4 on the driver's command shape (20 flushed ticks), alternated
for r in 1 2 3; do for c in 2 3 4; do
  HB_CHAIN_CHUNKS=$c timeout 300 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > /tmp/b.json 2>/dev/null
  python -c "import json;d=json.loads(open('/tmp/b.json').read().strip().splitlines()[-1]);print('chunks=$c', round(d['value']), round(d['ms_per_step'],4), d['clocks']['sm_mhz'])"
done; done
