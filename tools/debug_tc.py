"""Per-block gradient comparison of the GPU regression tile vs the FP64 oracle (debug aid)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402

import oracle_api  # noqa: E402
import paper_2211_17005_b200 as hcva  # noqa: E402
from paper_2211_17005_b200 import regression as rg  # noqa: E402


def main(d=12, u=32, rows=700, head=False):
    R = oracle_api.restatement()
    rng = np.random.default_rng(3)
    x = rng.standard_normal((rows, d))
    y = np.abs(np.sin(x[:, 0]) + 0.1 * rng.standard_normal(rows))
    t = hcva.TrainConfig()
    t.width, t.hidden_layers = u, 2
    p = R.init_network(d, 2, u, R.key(5))
    p[-1] = 0.2
    lo, go = R.loss(p, x, y, 2, u, 0, head)
    lg, gg = rg.quadratic_loss(t, p, x, y, head)
    print("loss", lg, lo)
    names = [("W0", u * d), ("b0", u), ("W1", u * u), ("b1", u), ("w2", u), ("b2", 1), ("mu", 1)]
    off = 0
    for nm, n in names:
        a, b = gg[off:off + n], go[off:off + n]
        err = np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30)
        print(f"{nm:3s} n={n:5d} relerr={err:.3e} gpu[:3]={a[:3]} ref[:3]={b[:3]}")
        off += n


if __name__ == "__main__":
    for d, u, rows, head in ((12, 32, 700, False), (12, 32, 700, True), (21, 64, 1000, False), (5, 16, 130, True),
                             (64, 64, 4096, False)):
        print(f"--- d={d} u={u} rows={rows} head={head}")
        main(d, u, rows, head)
