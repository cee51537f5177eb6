"""K4b column-tile width sweep: the planner's pick (auto) against forced widths (HB_PP_NB), zero data."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib  # noqa: E402

L = _lib.lib()
shapes = [(192, 32, 7500, 1, 0), (192, 32, 7500, 1, 1), (192, 32, 7500, 2, 0), (192, 32, 3750, 1, 2), (192, 32, 1875, 1, 2),
          (64, 64, 7500, 1, 0), (64, 64, 7500, 1, 1), (64, 64, 1875, 1, 2), (192, 64, 1875, 1, 1), (192, 64, 469, 1, 2)]
nb = os.environ.get("HB_PP_NB", "auto")
for P, c, l, s, r in shapes:
    ms = C.c_float()
    rc = L.hb_bench_conv_k(P, c, c, l, s, r, 1, 20, C.byref(ms))
    print(f"{nb:>4} P={P:3d} C={c} L={l:4d} s={s} res={r}: " + (f"{ms.value*1e3:7.1f} us" if rc == 0 else "n/a"), flush=True)
