"""Exercise hcva_diag_tc_gemm over its operand-layout variants (debug aid)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2211_17005_b200 as hcva  # noqa: E402
from paper_2211_17005_b200 import _lib  # noqa: E402

L = _lib.lib()
L.hcva_diag_tc_gemm.argtypes = [C.c_void_p] + [C.c_int] * 4 + [C.c_void_p] * 3
rng = np.random.default_rng(0)
for M, N, K in ((128, 32, 16), (64, 32, 128), (128, 64, 64), (64, 48, 128)):
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    for var, name in enumerate(("kmajor", "kmajor-sw128", "a-mn", "b-mn", "both-mn", "a-mn-sw", "b-mn-sw", "both-mn-sw")):
        D = np.zeros((M, N), dtype=np.float32)
        rc = L.hcva_diag_tc_gemm(hcva.context().handle, M, N, K, var, A.ctypes.data, B.ctypes.data, D.ctypes.data)
        err = np.max(np.abs(D - ref)) / np.max(np.abs(ref))
        print(M, N, K, f"{name:13s}", "rc", rc, "relerr %.2e" % err, "D[0,:3]", D[0, :3], "ref", ref[0, :3])
