"""Per-shape conv kernel throughput (zero data, back-to-back launches)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib  # noqa: E402

L = _lib.lib()
P = int(sys.argv[1]) if len(sys.argv) > 1 else 64
shapes = [(c, c, l, s, r) for (c, l, s, r) in [(32, 7500, 1, 0), (32, 7500, 1, 1), (32, 7500, 2, 0), (32, 3750, 1, 1),
                                               (64, 7500, 1, 0), (64, 7500, 1, 1), (64, 3750, 2, 0), (64, 1875, 1, 1),
                                               (128, 3750, 1, 0), (128, 938, 1, 1), (256, 938, 1, 0), (256, 469, 1, 1)]]
shapes += [(32, 64, 1875, 1, 0), (64, 128, 938, 1, 0), (128, 256, 469, 1, 0)]
for (ci, co, l, s, r) in shapes:
    ms = C.c_float()
    _lib.check(L.hb_bench_conv(P, ci, co, l, s, r, 20, C.byref(ms)))
    lout = -(-l // s)
    fl = 2 * ci * co * 16 * lout * P
    tiles = P * -(-lout // 128) * max(1, -(-co // 256))
    print(f"P={P:4d} cin={ci:4d} cout={co:4d} L={l:5d} s={s} res={r}: {ms.value*1e3:8.1f} us "
          f"{fl/ms.value/1e9:7.1f} TF/s  tiles/CTA={tiles/148:.1f}  us/tile={ms.value*1e3/(tiles/148):.2f}")
