#!/bin/bash
# K4c with the ensemble aggregation fused in (HB_CHAIN_AGG=1, default) vs the separate aggregate kernel
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_parity_timed_gpu.py tests/test_chain_fuzz_gpu.py tests/test_engine_gpu.py tests/test_parallel_gpu.py tests/test_runtime_gpu.py -m gpu -x -q -p no:cacheprovider 2>&1 | tail -3
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
AB_ROUNDS=6 timeout 300 python tools/abtick.py "HB_CHAIN_AGG=0" "HB_CHAIN_AGG=1" 2>&1 | tail -2
AB_ROUNDS=6 AB_P=16 timeout 300 python tools/abtick.py "HB_CHAIN_AGG=0" "HB_CHAIN_AGG=1" 2>&1 | tail -2
timeout 600 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/agg_bench20.json 2> gpurun_out/agg_bench20.err; echo "bench20 rc=$?"
HB_CHAIN_AGG=0 timeout 600 python bench.py --steps 20 --warmup 5 --no-extras --no-cpu-baseline > gpurun_out/agg0_bench20.json 2> gpurun_out/agg0_bench20.err; echo "bench20 agg0 rc=$?"
python - <<'PY'
import json
for f in ("gpurun_out/agg0_bench20.json", "gpurun_out/agg_bench20.json"):
    d = json.loads(open(f).read().strip().splitlines()[-1])
    print(f, round(d["value"]), round(d["ms_per_step"], 4), d["e2e"]["value"], d["gpu_launches"], d["clocks"]["sm_mhz"], d["parity"]["ok"])
PY
