"""Measure the kind::tf32 tcgen05 MMA rate per shape (hcva_diag_tc_rate; profiling aid)."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2211_17005_b200 as hcva  # noqa: E402
from paper_2211_17005_b200 import _lib  # noqa: E402

L = _lib.lib()
L.hcva_diag_tc_rate.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_double)]
ctx = hcva.context()
for M, N in ((128, 64), (128, 128), (128, 256), (64, 64), (64, 32), (128, 32), (128, 16)):
    for iters in (256, 4096):
        v = C.c_double()
        _lib.check(L.hcva_diag_tc_rate(ctx.handle, M, N, iters, C.byref(v)))
        print(f"M={M:3d} N={N:3d} iters={iters:5d}: {v.value:8.1f} TFLOP/s (tf32)")
