"""K4b shortcut cost per shape: none / identity / maxpool (P rows), with role-cycle counters under HB_PP_DBG=16."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib  # noqa: E402

L = _lib.lib()
for P, c, l in [(192, 32, 3750), (192, 32, 1875), (192, 64, 938), (64, 64, 3750), (64, 64, 938)]:
    for r in (0, 1, 2):
        ms = C.c_float()
        rc = L.hb_bench_conv_k(P, c, c, l, 1, r, 1, 20, C.byref(ms))
        print(f"P={P} C={c} L={l} res={r}: " + (f"{ms.value*1e3:7.1f} us" if rc == 0 else f"rc={rc}"), flush=True)
