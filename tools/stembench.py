"""Stem (K3) launch time on zero data: python tools/stembench.py  (HB_STEM=0 selects the Toeplitz kernel)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib  # noqa: E402

L = _lib.lib()
shapes = [(3, 64, 32, 4), (1, 64, 64, 2), (1, 64, 16, 8), (1, 64, 8, 1), (1, 64, 128, 1), (3, 64, 128, 1),
          (1, 1024, 32, 4)]
if len(sys.argv) > 1:
    shapes = [tuple(int(v) for v in sys.argv[1].split(','))]
for (G, Pm, cout, q) in shapes:
    ms = C.c_float()
    rc = L.hb_bench_stem(G, Pm, 7500, cout, q, 50, C.byref(ms))
    n = G * Pm
    gbs = n * 7500 * cout * 2 / ms.value / 1e6 if rc == 0 else 0
    print(f"G={G} Pm={Pm} C={cout:3d} Q={q}: " + (f"{ms.value*1e3:7.1f} us  {gbs:7.0f} GB/s out" if rc == 0 else f"rc={rc} {L.hb_last_error(None)}"),
          flush=True)
