"""c3 (full 60-member zoo, 100 beds): eager per-launch times grouped by kernel kind and layer width."""
import collections
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200.engine import EnsembleEngine  # noqa: E402
from paper_2008_04063_b200.zoo import Selector, holmes_zoo  # noqa: E402

KIND = {0: "ingest", 1: "stem", 2: "K4", 3: "aggregate", 4: "advance", 5: "K4b"}
zoo = holmes_zoo()
P = int(sys.argv[1]) if len(sys.argv) > 1 else 100
eng = EnsembleEngine(zoo, Selector.ones(60), P, hop=250)
eng.ingest(np.random.default_rng(0).standard_normal((P, 3, 7500)).astype(np.float32))
s = torch.cuda.Stream()
eng.profile_tick(s.cuda_stream)
k, ms, fl, by = eng.profile_tick(s.cuda_stream)
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for i in range(len(k)):
    a = agg[KIND[int(k[i])]]
    a[0] += 1
    a[1] += ms[i]
    a[2] += fl[i]
tot = ms.sum()
for name, (n, t, f) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{name:10s} {n:4d} launches {t:8.2f} ms ({t / tot * 100:5.1f}%) {f / max(t, 1e-9) / 1e9:7.1f} TF/s")
print(f"eager total {tot:.2f} ms; graph tick {eng.time_tick(3) * 1e3:.2f} ms")
# the slowest launches
order = np.argsort(-ms)[:15]
for i in order:
    print(f"  #{i:4d} {KIND[int(k[i])]:5s} {ms[i] * 1e3:8.1f} us {fl[i] / ms[i] / 1e9 if ms[i] > 0 else 0:7.1f} TF/s {fl[i] / 1e9:8.2f} GFLOP")
order = np.argsort(-ms)[:25]
print("top launches: index kind ms TF/s GFLOP MB")
for i in order:
    print(f"{i:5d} {KIND[int(k[i])]:6s} {ms[i]:7.3f} {fl[i] / max(ms[i], 1e-9) / 1e9:7.1f} {fl[i] / 1e9:8.1f} {by[i] / 1e6:8.1f}")
