"""K4b timing under HB_PP_DBG knobs (one process per setting: the knob is read per plan).
usage: HB_PP_DBG=<bits> python tools/ppdbg_matrix.py"""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib  # noqa: E402

L = _lib.lib()
out = []
for P in (192, 1024):
    for (ci, co, l, s, r) in [(32, 32, 7500, 1, 0), (32, 32, 7500, 2, 0), (64, 64, 7500, 1, 0), (64, 64, 1875, 2, 0)]:
        ms = C.c_float()
        rc = L.hb_bench_conv_k(P, ci, co, l, s, r, 1, 20, C.byref(ms))
        lout = -(-l // s)
        fl = 2 * ci * co * 16 * lout * P
        out.append(f"P={P} {ci}->{co} L={l} s={s}: " + (f"{ms.value*1e3:8.1f} us {fl/ms.value/1e9:7.1f} TF/s" if rc == 0 else f"rc {rc}"))
print(f"dbg={os.environ.get('HB_PP_DBG', '0')}: " + " | ".join(out))
