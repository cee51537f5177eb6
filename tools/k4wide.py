"""K4 on the full zoo's wide layers (zero data, back-to-back launches): python tools/k4wide.py [P]"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib  # noqa: E402

L = _lib.lib()
P = int(sys.argv[1]) if len(sys.argv) > 1 else 100
iters = int(os.environ.get("K4W_ITERS", "10"))
shapes = [(128, 128, 3750, 1, 1), (256, 256, 1875, 1, 1), (256, 256, 1875, 2, 2), (512, 512, 469, 1, 1),
          (512, 512, 938, 1, 1), (1024, 1024, 118, 1, 1), (1024, 1024, 59, 1, 1), (1024, 1024, 30, 1, 1),
          (512, 1024, 235, 1, 0)]
if os.environ.get("K4W_SHAPES"):
    shapes = [tuple(int(x) for x in s.split(":")) for s in os.environ["K4W_SHAPES"].split(",")]
for (ci, co, l, s, r) in shapes:
    lout = -(-l // s)
    fl = 2 * ci * co * 16 * lout * P
    ms = C.c_float()
    rc = L.hb_bench_conv_k(P, ci, co, l, s, r, 0, iters, C.byref(ms))
    print(f"P={P} {ci}->{co} L={l} s={s} res={r}: " + (f"{ms.value*1e3:8.1f} us {fl/ms.value/1e9:7.1f} TF/s" if rc == 0 else f"rc={rc}"), flush=True)
