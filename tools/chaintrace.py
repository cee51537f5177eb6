"""Per-layer timeline of one K4c chain launch (HB_CHAIN_PROF=1): for every chain
layer, when its items were pulled / became ready / were published, and how
long items waited for dependencies.  usage: python tools/chaintrace.py [P] [out.npz]"""
import ctypes as C
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
os.environ.setdefault("HB_CHAIN_PROF", "1")
from paper_2008_04063_b200 import _lib  # noqa: E402
from paper_2008_04063_b200.engine import EnsembleEngine  # noqa: E402
from paper_2008_04063_b200.zoo import Selector, holmes_zoo  # noqa: E402

P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
idx = [10, 13, 30, 50]
eng = EnsembleEngine(holmes_zoo(), Selector.from_indices(60, idx), P, hop=250)
eng.ingest(np.random.default_rng(0).standard_normal((P, 3, 7500)).astype(np.float32))
for _ in range(3):
    eng.time_tick(1)
cap = 1 << 20
tr = np.zeros((cap, 5), np.uint64)
items = np.zeros(cap, np.int32)
n = _lib.lib().hb_chain_trace(eng._h, tr.ctypes.data_as(C.c_void_p), items.ctypes.data_as(C.c_void_p), cap)
tr, items = tr[:n].astype(np.int64), items[:n]
if len(sys.argv) > 2:
    np.savez(sys.argv[2], trace=tr, items=items)
t0 = tr[:, 0].min()
pull, wdone, ready = (tr[:, 0] - t0) / 1e3, (tr[:, 1] - t0) / 1e3, (tr[:, 2] - t0) / 1e3
done = (np.maximum(tr[:, 3], tr[:, 4]) - t0) / 1e3
layer = items >> 22
print(f"items {n}; launch span {done.max():.1f} us (first pull -> last publish)")
print(f"{'layer':>5} {'items':>6} {'pull0':>8} {'pullN':>8} {'done0':>8} {'doneN':>8} {'w/item':>8} {'dw/item':>8} {'lat/item':>8}")
for li in sorted(set(layer.tolist())):
    m = layer == li
    ww = wdone[m] - pull[m]
    dw = ready[m] - wdone[m]
    lat = done[m] - ready[m]
    print(f"{li:5d} {m.sum():6d} {pull[m].min():8.1f} {pull[m].max():8.1f} {done[m].min():8.1f} {done[m].max():8.1f} "
          f"{ww.mean():8.2f} {dw.mean():8.2f} {lat.mean():8.2f}")
d = np.diff(np.sort(tr[:, 0]))
print("globaltimer resolution (smallest nonzero step between pulls, ns):", int(d[d > 0].min()) if (d > 0).any() else None)
