#!/bin/bash
# Round-2 verification of the restored tree: full GPU suite, smoke, bench (patient, member, reference arm).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/gpu.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider --durations=20 > gpurun_out/gputests.log 2>&1; echo "rc=$?" >> gpurun_out/gputests.log
tail -30 gpurun_out/gputests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
tail -3 gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -3 gpurun_out/bench_default.err
timeout 600 python bench.py --mode member --steps 20 --warmup 3 --no-cpu-baseline > gpurun_out/bench_member.json 2> gpurun_out/bench_member.err; echo "member rc=$?"
tail -3 gpurun_out/bench_member.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err; echo "ref rc=$?"
tail -3 gpurun_out/bench_ref.err
