"""Role cycle counters of the K4c chain launch (run with HB_CHAIN=1 HB_CHAIN_PROF=1).
usage: python tools/chainprof.py [P] [idx,idx,...]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib  # noqa: E402
from paper_2008_04063_b200.engine import EnsembleEngine  # noqa: E402
from paper_2008_04063_b200.zoo import Selector, holmes_zoo  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
idx = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [10, 13, 30, 50]
eng = EnsembleEngine(holmes_zoo(), Selector.from_indices(60, idx), P, hop=250)
eng.ingest(np.random.default_rng(0).standard_normal((P, 3, 7500)).astype(np.float32))
print("graph tick ms", eng.time_tick(10))
buf = np.zeros((148, 16), np.uint64)
n = _lib.lib().hb_chain_profile(eng._h, buf.ctypes.data_as(C.c_void_p), 148)
if n <= 0:
    sys.exit("no chain profile (HB_CHAIN=1 HB_CHAIN_PROF=1?)")
b = buf[:n].astype(np.float64) / 1.9e3  # cycles -> us at ~1.9 GHz
names = ["prod_dep", "prod_w", "prod_stage", "prod_total", "items", "mma_w", "mma_acc", "mma_stage", "mma_total",
         "epi_accwait", "epi_total"]
print("cta " + " ".join(f"{x:>10s}" for x in names))
for r in range(n):
    row = b[r].copy()
    row[4] = buf[r, 4]
    print(f"{r:3d} " + " ".join(f"{v:10.1f}" for v in row[:11]))
print("mean " + " ".join(f"{v:10.1f}" for v in b[:, :11].mean(0)))
