#!/bin/bash
# Round evidence: GPU tests + smoke, conv DRAM traffic per tick (both conv kernels), bench line,
# launch list, full ncu captures of K4b (largest c2 launch), K4 (head layer), window and sweep kernels.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:conv_ --csv --log-file gpurun_out/conv_traffic.csv python tools/prof1.py 10,13,30,50 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/conv_traffic.csv profiles/ncu_conv_summary.json > gpurun_out/conv_traffic.json 2>&1
cp profiles/ncu_conv_summary.json gpurun_out/ncu_conv_summary.json
timeout 900 python bench.py --steps 100 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --profile-only --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_pp -s 0 -c 1 \
  -o gpurun_out/prof_pp -f python tools/prof1.py 10,13,30,50 > gpurun_out/ncu_pp.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:conv_tc -s 0 -c 1 \
  -o gpurun_out/prof_conv -f python tools/prof1.py 10,13,30,50 > gpurun_out/ncu_conv.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:ingest_window -s 1 -c 1 \
  -o gpurun_out/prof_window -f python tools/prof1.py 10,13,30,50 > gpurun_out/ncu_window.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:sweep_auc -c 1 \
  -o gpurun_out/prof_sweep -f python tools/sweep1.py > gpurun_out/ncu_sweep.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 1 --steps 20 --warmup 3 --no-cpu-baseline --no-extras > gpurun_out/bench_torchrun.json 2> gpurun_out/bench_torchrun.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -2 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log; head -c 600 gpurun_out/bench.json; echo; head -12 gpurun_out/conv_traffic.json
