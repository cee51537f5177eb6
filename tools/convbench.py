import sys, ctypes as C
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2008_04063_b200 import _lib
L = _lib.lib()
shapes = [(64, c, c, l, s, r) for (c, l, s, r) in [(32,7500,1,0),(32,7500,1,1),(64,7500,1,0),(64,7500,1,1),(64,3750,2,0),(128,3750,1,0),(256,1875,1,0)]]
shapes += [(64, 64, 128, 7500, 1, 0), (64, 64, 256, 3750, 1, 0), (64, 32, 64, 7500, 1, 0), (256, 32, 32, 7500, 1, 0)]
for (P, ci, co, l, s, r) in shapes:
    ms = C.c_float()
    _lib.check(L.hb_bench_conv(P, ci, co, l, s, r, 20, C.byref(ms)))
    lout = -(-l // s)
    fl = 2 * ci * co * 16 * lout * P
    tiles = P * -(-lout // 128) * max(1, -(-co // 256))
    print(f"P={P:4d} cin={ci:4d} cout={co:4d} L={l:5d} s={s} res={r}: {ms.value*1e3:8.1f} us {fl/ms.value/1e9:7.1f} TF/s  tiles/CTA={tiles/148:.1f}  us/tile={ms.value*1e3/(tiles/148):.2f}")
