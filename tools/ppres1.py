"""One K4b maxpool-shortcut layer shape, back-to-back (ncu target): 192 rows, 32 channels, L 3750."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2008_04063_b200 import _lib  # noqa: E402

ms = C.c_float()
_lib.check(_lib.lib().hb_bench_conv_k(192, 32, 32, 3750, 1, int(sys.argv[1]) if len(sys.argv) > 1 else 2, 1, 3,
                                      C.byref(ms)))
print(ms.value)
