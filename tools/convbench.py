"""Per-shape conv kernel throughput (zero data, back-to-back launches).

python tools/convbench.py [P ...] [--pp]: with --pp every shape K4b supports is
timed on both kernels (K4 = positions on M, K4b = polyphase) side by side.
"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib  # noqa: E402

L = _lib.lib()
args = [a for a in sys.argv[1:] if not a.startswith("--")]
both = "--pp" in sys.argv
Ps = [int(a) for a in args] or ([64, 512] if both else [64])
shapes = [(c, c, l, s, r) for (c, l, s, r) in [(32, 7500, 1, 0), (32, 7500, 1, 1), (32, 7500, 2, 0), (32, 3750, 1, 1),
                                               (32, 3750, 2, 0), (32, 1875, 1, 1),
                                               (64, 7500, 1, 0), (64, 7500, 1, 1), (64, 3750, 2, 0), (64, 1875, 1, 1),
                                               (64, 938, 1, 1), (64, 938, 2, 0), (64, 469, 1, 1),
                                               (16, 7500, 1, 1), (16, 3750, 2, 0),
                                               (128, 3750, 1, 0), (128, 938, 1, 1), (256, 938, 1, 0), (256, 469, 1, 1)]]
shapes += [(32, 64, 1875, 1, 0), (16, 32, 1875, 1, 0), (64, 128, 938, 1, 0), (128, 256, 469, 1, 0)]


def bench(P, ci, co, l, s, r, kind):
    ms = C.c_float()
    rc = L.hb_bench_conv_k(P, ci, co, l, s, r, kind, 20, C.byref(ms))
    if rc != 0:
        return None
    return ms.value


for P in Ps:
    for (ci, co, l, s, r) in shapes:
        lout = -(-l // s)
        fl = 2 * ci * co * 16 * lout * P
        t_tc = bench(P, ci, co, l, s, r, 0)
        line = f"P={P:4d} cin={ci:4d} cout={co:4d} L={l:5d} s={s} res={r}:"
        line += f"  K4 {t_tc*1e3:8.1f} us {fl/t_tc/1e9:7.1f} TF/s" if t_tc else "  K4 n/a"
        if both and L.hb_conv_kind(ci, co, s, 0) == 1:
            t_pp = bench(P, ci, co, l, s, r, 1)
            line += (f" | K4b {t_pp*1e3:8.1f} us {fl/t_pp/1e9:7.1f} TF/s  x{t_tc/t_pp:.2f}" if t_pp and t_tc
                     else " | K4b failed")
        print(line, flush=True)
