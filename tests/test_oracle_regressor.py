"""Pin the FP64 regression restatement (oracle/regress_oracle.c) with the
reference's own regressor tests (proj/tests/test_regressor.cpp), restated.
The reference regressor cannot be compiled here (Eigen is absent), so these
analytic / behavioural checks are what anchors the oracle."""
import numpy as np
import pytest

import oracle_api


@pytest.fixture(scope="module")
def R():
    return oracle_api.restatement()


class Stream:
    """Sequential draws of one oracle stream (RandomStream::next_*)."""

    def __init__(self, R, key):
        self.R, self.key, self.j = R, key, 0

    def normal(self, n=1):
        v = self.R.normals(self.key, self.j, n)
        self.j += n
        return v

    def uniform(self, n=1):
        v = self.R.uniforms(self.key, self.j, n)
        self.j += n
        return v


def fd_check(R, p, x, y, hidden, width, act, head):
    _, g = R.loss(p, x, y, hidden, width, act, head)
    worst = 0.0
    for s in range(p.size):
        h = 1e-6 * max(1.0, abs(p[s]))
        q = p.copy()
        q[s] += h
        lp = R.loss(q, x, y, hidden, width, act, head, grads=False)
        q[s] -= 2 * h
        lm = R.loss(q, x, y, hidden, width, act, head, grads=False)
        fd = (lp - lm) / (2 * h)
        scale = max(abs(fd), abs(g[s]), 1e-8)
        worst = max(worst, abs(fd - g[s]) / scale)
    return worst


@pytest.mark.parametrize("act", [0, 1, 2])
def test_gradients_match_finite_differences(R, act):
    """test_regressor.cpp:68-110 (tanh, sigmoid, softplus; rel 1e-5)."""
    p = R.init_network(4, 2, 6, R.key(11))
    p[-1] = 0.1
    ds = Stream(R, R.key(12))
    x = np.zeros((10, 4))
    y = np.zeros(10)
    for i in range(10):
        x[i] = ds.normal(4)
        y[i] = ds.normal()[0]
    assert fd_check(R, p, x, y, 2, 6, act, False) < 1e-5


def test_positive_head_gradients(R):
    """test_regressor.cpp:112-138."""
    p = R.init_network(3, 2, 6, R.key(21))
    p[-1] = 0.05
    ds = Stream(R, R.key(22))
    x = np.zeros((16, 3))
    y = np.zeros(16)
    for i in range(16):
        x[i] = ds.normal(3)
        y[i] = abs(ds.normal()[0])
    assert fd_check(R, p, x, y, 2, 6, 0, True) < 1e-5


def test_refit_solves_ridge_normal_equations(R):
    """test_regressor.cpp:167-202: width-1 hidden layer vs the hand 2x2 solve (1e-10)."""
    p = R.init_network(1, 1, 1, R.key(31))
    p[-1] = 0.2
    ds = Stream(R, R.key(32))
    x = np.zeros((40, 1))
    y = np.zeros(40)
    for i in range(40):
        x[i, 0] = ds.normal()[0]
        y[i] = 0.8 * x[i, 0] + 0.1 * ds.normal()[0]
    q = R.refit(p, x, y, 1, 1, 1e-8)
    w0, b0 = p[0], p[1]
    hid = np.tanh(w0 * x[:, 0] + b0)
    shh, sh1, s11 = np.sum(hid * hid), np.sum(hid), 40.0
    shy, s1y = np.sum(hid * (y - 0.2)), np.sum(y - 0.2)
    lam = 1e-8 * (shh + s11) / 2
    det = (shh + lam) * (s11 + lam) - sh1 * sh1
    w_hand = ((s11 + lam) * shy - sh1 * s1y) / det
    b_hand = ((shh + lam) * s1y - sh1 * shy) / det
    assert q[2] == pytest.approx(w_hand, rel=1e-10)
    assert q[3] == pytest.approx(b_hand, rel=1e-10)


def test_refit_never_raises_mse(R):
    """test_regressor.cpp:204-226."""
    for inst in range(20):
        p = R.init_network(3, 2, 8, R.key(777, inst))
        p[-1] = 0.1 * inst
        ds = Stream(R, R.key(777, 1000 + inst))
        x = np.zeros((64, 3))
        y = np.zeros(64)
        for i in range(64):
            x[i] = ds.normal(3)
            y[i] = np.sin(x[i, 0]) + 0.3 * ds.normal()[0]
        before = R.loss(p, x, y, 2, 8, grads=False)
        after = R.loss(R.refit(p, x, y, 2, 8), x, y, 2, 8, grads=False)
        assert after <= before + 1e-8 * max(1.0, before)


def test_constant_labels_fit_to_mean(R):
    """test_regressor.cpp:241-255."""
    ds = Stream(R, R.key(51))
    x = ds.normal(512 * 2).reshape(512, 2)
    y = np.full(512, 0.7)
    init = R.init_network(2, 2, 16, R.key(7))
    init[-1] = y.mean()
    _, rep = R.train_base(x, y, init, 2, 16, 8, 8)
    assert rep["best_loss"] <= 1e-6


def test_best_tracking_exact(R):
    """test_regressor.cpp:257-281."""
    ds = Stream(R, R.key(61))
    x = np.zeros((256, 2))
    y = np.zeros(256)
    for i in range(256):
        x[i] = ds.normal(2)
        y[i] = x[i, 0] ** 2 + 0.2 * ds.normal()[0]
    init = R.init_network(2, 2, 16, R.key(7))
    init[-1] = y.mean()
    best, rep = R.train_base(x, y, init, 2, 16, 4, 10)
    assert rep["best_loss"] == pytest.approx(rep["epoch_losses"].min(), rel=1e-15)
    assert R.loss(best, x, y, 2, 16, head=True, grads=False) == pytest.approx(rep["best_loss"], rel=1e-12)


def test_toy_regression_noise_floor(R):
    """test_regressor.cpp:283-304: out-of-sample MSE within 10% of the noise variance."""
    ds = Stream(R, R.key(71))
    n = 10000
    x, xt, y, yt = np.zeros((n, 1)), np.zeros((n, 1)), np.zeros(n), np.zeros(n)
    for i in range(n):
        x[i, 0] = 2 * ds.uniform()[0] - 1
        y[i] = x[i, 0] ** 2 + 0.1 * ds.normal()[0]
        xt[i, 0] = 2 * ds.uniform()[0] - 1
        yt[i] = xt[i, 0] ** 2 + 0.1 * ds.normal()[0]
    init = R.init_network(1, 2, 32, R.key(7))
    init[-1] = y.mean()
    best, _ = R.train_base(x, y, init, 2, 32, 25, 40)
    oos = R.loss(best, xt, yt, 2, 32, head=True, grads=False)
    assert 0.9 * 0.01 < oos < 1.1 * 0.01


def test_backward_learn_n1_is_train_base_and_deterministic(R):
    """test_regressor.cpp:306-335 and :379-415 (determinism)."""
    ds = Stream(R, R.key(81))
    x = np.zeros((128, 2))
    y = np.zeros(128)
    for i in range(128):
        x[i] = ds.normal(2)
        y[i] = x[i, 0] + 0.1 * ds.normal()[0]
    src = lambda i: (x, y, 0)  # noqa: E731
    a = R.backward_learn(1, src, 7, 2, 8, 4, 6)
    b = R.backward_learn(1, src, 7, 2, 8, 4, 6)
    mean, scale = R.fit_scaler(x, 0)
    init = R.init_network(2, 2, 8, R.key(7, 0xBEEF, 1))
    init[-1] = y.mean()
    best, rep = R.train_base((x - mean) / scale, y, init, 2, 8, 4, 6)
    assert np.array_equal(a[1][0], best) and np.array_equal(a[1][0], b[1][0])
    assert rep["best_loss"] == a[1][3]["best_loss"]
