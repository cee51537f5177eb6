"""64-channel stride-2 K4b layers (164 KB weight image): time per forced column tile width (HB_PP_NB)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib  # noqa: E402

L = _lib.lib()
for P, c, l in [(192, 64, 3750), (192, 64, 1875), (192, 64, 938), (64, 64, 3750), (64, 64, 938)]:
    ms = C.c_float()
    rc = L.hb_bench_conv_k(P, c, c, l, 2, 0, 1, 20, C.byref(ms))
    print(f"NB={os.environ.get('HB_PP_NB', 'auto')} P={P} C={c} L={l} s2: " + (f"{ms.value*1e3:7.1f} us" if rc == 0 else f"rc={rc}"),
          flush=True)
