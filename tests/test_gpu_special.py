"""Accuracy of the device special functions behind the normal transform
(paper_2211_17005_b200/csrc/normal.cuh) against correctly rounded mpmath values
(tests/golden/special.npz).  libdevice's erfc is documented at <= 4 ulp and
glibc's at ~1 ulp; the custom erfc is held to 4 ulp, exp to 2 ulp."""
import ctypes as C

import numpy as np
import pytest

import oracle_api
import paper_2211_17005_b200 as hcva
from paper_2211_17005_b200 import _lib

pytestmark = pytest.mark.gpu


def special(fn, x):
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros_like(x)
    _lib.check(_lib.lib().hcva_diag_special(hcva.context().handle, fn, x.ctypes.data_as(C.c_void_p), x.size,
                                            out.ctypes.data_as(C.c_void_p)))
    return out


def ulps(a, b):
    return np.abs(a - b) / np.spacing(np.abs(b))


def test_erfc_fast_within_4_ulp():
    z = np.load(f"{oracle_api.ROOT}/tests/golden/special.npz")
    got = special(0, z["erfc_x"])
    u = ulps(got, z["erfc_y"])
    print(f"erfc: max {u.max():.0f} ulp, mean {u.mean():.3f}, exact {np.mean(u == 0):.3f}")
    assert u.max() <= 4


def test_exp_neg_within_2_ulp():
    z = np.load(f"{oracle_api.ROOT}/tests/golden/special.npz")
    got = special(1, z["exp_x"])
    u = ulps(got, z["exp_y"])
    print(f"exp: max {u.max():.0f} ulp, mean {u.mean():.3f}")
    assert u.max() <= 2
    e = special(3, z["erfc_x"])
    want = np.exp(-z["erfc_x"] ** 2)  # numpy rounds x^2 first: ~|x|^2 ulp of slack
    assert np.max(np.abs(e / want - 1)) < 1e-14


def test_normal_transform_matches_k0():
    """hcva_rng_draw(kind=2) and the diag entry agree bit for bit (same device code)."""
    s = hcva.RandomStream(11)
    u = s.uniforms(4096)
    assert np.array_equal(special(2, u), hcva.RandomStream(11).normals(4096))
