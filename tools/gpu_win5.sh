#!/bin/bash
# window kernel: parity + ncu launch durations per window misalignment (hop 248: A=0; 250: 0,2; 251: 3,2,1,0)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_parity_timed_gpu.py -k "window or c2_64 or north_star or HB_WIN" -m gpu -q -p no:cacheprovider -x > gpurun_out/win_tests.log 2>&1; echo "rc=$?" >> gpurun_out/win_tests.log
tail -2 gpurun_out/win_tests.log
for nb in 1 3 4; do HB_WIN_NB=$nb timeout 900 python -m pytest tests/test_parity_timed_gpu.py -k "window" -m gpu -q -p no:cacheprovider -x 2>&1 | tail -1; done
for P in 1024 64; do
for H in 248 251; do
for V in "HB_WIN_NB=2" "HB_WIN_NB=4" "HB_WIN_NB=1" "HB_WIN_NB=3"; do
  echo -n "P=$P hop=$H $V: "
  env $V timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none \
    -k regex:ingest_window -s 1 -c 8 --csv python tools/win_tick.py $P $H 10 2>/dev/null | grep gpu__time_duration | \
    awk -F'","' '{gsub(/"/,"",$NF); printf "%s ", $NF}'; echo
done
done
done
