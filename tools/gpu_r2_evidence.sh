#!/bin/bash
# Round-2 evidence on the K4c chain tick: bench lines, ncu launch list, ncu DRAM traffic + full capture
# of the chain launch, compute-sanitizer on the chain.
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/gpu.txt 2>&1
timeout 900 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
timeout 600 python bench.py --steps 20 --warmup 5 --no-extras > gpurun_out/r02_bench20.json 2> gpurun_out/r02_bench20.err; echo "bench20 rc=$?"
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/r02_ref.json 2> gpurun_out/r02_ref.err; echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv \
  --log-file gpurun_out/r02_launches.csv python bench.py --steps 3 --warmup 3 --profile-only --no-cpu-baseline > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r02_launches.csv > gpurun_out/r02_launches_summary.txt; cat gpurun_out/r02_launches_summary.txt
timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:"conv_|chain_" --csv --log-file gpurun_out/conv_traffic.csv python tools/prof1.py 10,13,30,50 > /dev/null 2>&1
python tools/ncu_traffic.py gpurun_out/conv_traffic.csv gpurun_out/ncu_conv_summary.json | head -12
timeout 900 ncu --set full --clock-control none --import-source on -k regex:chain_pp -c 1 \
  -o gpurun_out/prof_chain -f python tools/prof1.py 10,13,30,50 > gpurun_out/ncu_chain.log 2>&1
python tools/ncu_summary.py gpurun_out/prof_chain.ncu-rep > gpurun_out/r02_ncu_chain_summary.txt 2>&1
head -30 gpurun_out/r02_ncu_chain_summary.txt
{
timeout 900 compute-sanitizer --tool memcheck --print-limit 20 python -m pytest tests/test_parity_timed_gpu.py -x -q -p no:cacheprovider -k "c2_64 or chain_capped_grid" 2>&1 | tail -3
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_parity_timed_gpu.py -x -q -p no:cacheprovider -k "chain_capped_grid and 13" 2>&1 | tail -3
timeout 900 compute-sanitizer --tool synccheck --print-limit 10 python -m pytest tests/test_parity_timed_gpu.py -x -q -p no:cacheprovider -k "chain_capped_grid and 13" 2>&1 | tail -3
# the per-layer path (K4b with the all-warpgroup epilogue, K4, stems)
timeout 900 compute-sanitizer --tool racecheck --print-limit 10 python -m pytest tests/test_parity_timed_gpu.py -x -q -p no:cacheprovider -k "multi_tile_paths_forced and 6" 2>&1 | tail -3
timeout 900 compute-sanitizer --tool memcheck --print-limit 10 python -m pytest tests/test_engine_gpu.py -x -q -p no:cacheprovider -k "sliding or nonfinite" 2>&1 | tail -3
} > gpurun_out/r02_sanitizer.txt 2>&1
cat gpurun_out/r02_sanitizer.txt
