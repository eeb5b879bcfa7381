"""Golden values for the device special functions (tests/test_gpu_special.py):
erfc on [-6, 6] and exp on [-40, 0], correctly rounded from mpmath at 40 digits.
    python tests/golden/make_special.py
"""
import os

import mpmath as mp
import numpy as np

mp.mp.dps = 40
HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    rng = np.random.default_rng(7)
    xe = np.concatenate([np.linspace(-6, 6, 6001), rng.uniform(-6, 6, 4000), [0.0, 2.0, -2.0, 6.0, -6.0]])
    ye = np.array([float(mp.erfc(mp.mpf(float(x)))) for x in xe])
    xz = np.concatenate([np.linspace(-40, 0, 4001), rng.uniform(-40, 0, 2000)])
    yz = np.array([float(mp.exp(mp.mpf(float(x)))) for x in xz])
    np.savez_compressed(os.path.join(HERE, "special.npz"), erfc_x=xe, erfc_y=ye, exp_x=xz, exp_y=yz)


if __name__ == "__main__":
    main()
