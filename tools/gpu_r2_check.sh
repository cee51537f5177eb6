#!/bin/bash
# Round-2 check: parity suite + parallel tests + bench (patient, member, reference arm).
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_parity_timed_gpu.py tests/test_engine_gpu.py tests/test_parallel_gpu.py -m gpu -q -p no:cacheprovider -x > gpurun_out/parity.log 2>&1; echo "rc=$?" >> gpurun_out/parity.log
tail -4 gpurun_out/parity.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench20.json 2> gpurun_out/bench20.err; echo "bench rc=$?"
tail -3 gpurun_out/bench20.err
timeout 600 python bench.py --mode member --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_member.json 2> gpurun_out/bench_member.err; echo "member rc=$?"
tail -3 gpurun_out/bench_member.err
timeout 600 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
python - <<'PY'
import json
for f in ("bench20", "bench_member", "bench_ref"):
    try:
        d = json.load(open(f"gpurun_out/{f}.json"))
    except Exception as e:
        print(f, "unreadable", e); continue
    print(f, round(d["value"]), d["unit"], "ms/step", round(d["ms_per_step"], 4), "lat", d.get("latency_ms"))
    print("  parity", d.get("parity"))
    print("  e2e", {k: v for k, v in d["e2e"].items() if k != "api"})
    if "roofline" in d: print("  roof", d["roofline"]["achieved"], d["roofline"]["frac"], d["roofline"]["frac_of_sustained"])
    if "detail" in d:
        for k in ("beds_1024", "c3_full_zoo_100_beds", "nccl_reduce_ms"):
            if k in d["detail"]: print("  ", k, d["detail"][k])
PY
