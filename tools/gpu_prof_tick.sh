#!/bin/bash
timeout 300 python -m pytest tests/test_conv_gpu.py tests/test_conv_pp_gpu.py tests/test_engine_gpu.py -x -q -p no:cacheprovider -k "stem or engine or tick" 2>&1 | tail -2
timeout 300 python tools/layerprof.py > gpurun_out/layerprof.txt 2>&1; grep -E "stem|ingest" gpurun_out/layerprof.txt; tail -1 gpurun_out/layerprof.txt
timeout 300 python bench.py --steps 100 --warmup 5 --no-cpu-baseline --no-extras > gpurun_out/ab.json 2> gpurun_out/ab.err
python -c "import json;d=json.load(open('gpurun_out/ab.json'));print(round(d['value']), 'pw/s', round(d['ms_per_step'],4), 'ms e2e', round(d['e2e']['value']), d['clocks']['reasons'])"
