import ctypes as C, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib
L = _lib.lib()
for (ci, co, l) in [(32, 32, 7500), (64, 64, 7500)]:
    ms = C.c_float()
    _lib.check(L.hb_bench_conv(64, ci, co, l, 1, 0, 20, C.byref(ms)))
    print(ci, co, l, f"{ms.value*1e3:.1f} us", flush=True)
