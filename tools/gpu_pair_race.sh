#!/bin/bash
timeout 900 compute-sanitizer --tool racecheck --print-limit 3 python tests/_tick_worker.py /tmp/san.npz 2 250 1 3 15,16,17,36 2>&1 | head -60
