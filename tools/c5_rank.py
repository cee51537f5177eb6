"""Config c5 per rank: 8192 beds, the full zoo member-sharded 8 ways (FLOP-balanced);
runs the members of one rank's bin on this GPU (patient-chunked) and times the tick."""
import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import parallel
from paper_2008_04063_b200.engine import EnsembleEngine
from paper_2008_04063_b200.zoo import Selector, holmes_zoo
rank = int(sys.argv[1]) if len(sys.argv) > 1 else 3
P = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
zoo = holmes_zoo()
bins = parallel.member_bins(zoo, Selector.ones(60), 8)
sel = Selector.from_indices(60, bins[rank])
eng = EnsembleEngine(zoo, sel, P, hop=250)
t = eng.time_tick(reps=3)
f, _ = eng.tick_work()
print(f"c5 rank {rank}: {len(bins[rank])} members, {P} beds: tick {t*1e3:.1f} ms, {f/t/1e12:.0f} TFLOP/s", flush=True)
