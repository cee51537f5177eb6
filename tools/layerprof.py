"""Per-launch device times of one eagerly launched tick (events after every launch)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200.engine import EnsembleEngine  # noqa: E402
from paper_2008_04063_b200.zoo import Selector, holmes_zoo  # noqa: E402

KIND = {0: "ingest+window", 1: "stem", 2: "conv K4", 3: "aggregate", 4: "advance", 5: "conv K4b", 6: "chain K4c"}
zoo = holmes_zoo()
P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
idx = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [10, 13, 30, 50]
eng = EnsembleEngine(zoo, Selector.from_indices(60, idx), P, hop=250)
eng.ingest(np.random.default_rng(0).standard_normal((P, 3, 7500)).astype(np.float32))
s = torch.cuda.Stream()
for _ in range(3):
    eng.profile_tick(s.cuda_stream)
res = [eng.profile_tick(s.cuda_stream) for _ in range(5)]
k, fl, by = res[0][0], res[0][2], res[0][3]
ms = np.median([r[1] for r in res], axis=0)
for n in range(len(k)):
    tf = fl[n] / ms[n] / 1e9 if ms[n] > 0 else 0
    gb = by[n] / ms[n] / 1e6 if ms[n] > 0 else 0
    print(f"{n:3d} {KIND[int(k[n])]:14s} {ms[n]*1e3:8.1f} us {tf:7.1f} TF/s {gb:7.1f} GB/s  {fl[n]/1e9:8.2f} GFLOP")
print(f"eager total {ms.sum():.4f} ms; graph tick {eng.time_tick(20)*1e3:.4f} ms")
