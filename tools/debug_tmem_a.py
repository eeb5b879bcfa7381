"""Check the A-operand-in-tensor-memory tcgen05.mma (variant 8 of hcva_diag_tc_gemm,
used by k_sgd_tc / k_eval_tc) against the shared-memory K-major form (variant 0)."""
import ctypes as C, os, sys
sys.path.insert(0, "/root/repo")
import numpy as np
import paper_2211_17005_b200 as hcva
from paper_2211_17005_b200 import _lib
L = _lib.lib()
L.hcva_diag_tc_gemm.argtypes = [C.c_void_p] + [C.c_int] * 4 + [C.c_void_p] * 3
rng = np.random.default_rng(0)
for M, N, K in ((128, 32, 16), (128, 64, 64), (128, 128, 64)):
    A = rng.standard_normal((M, K)).astype(np.float32)
    B = rng.standard_normal((N, K)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    for var in (0, 8):
        D = np.zeros((M, N), dtype=np.float32)
        rc = L.hcva_diag_tc_gemm(hcva.context().handle, M, N, K, var, A.ctypes.data, B.ctypes.data, D.ctypes.data)
        err = np.max(np.abs(D - ref)) / np.max(np.abs(ref))
        print(M, N, K, var, "rc", rc, "relerr %.2e" % err, D[0, :3], ref[0, :3])
