"""Regression parity at the production shape of the paper case (C2): U = 64
hidden units, two hidden layers, d = 2*Cc + 3E - 1 = 45 inputs (dp = 48), so
the two-CTA tensor-core kernels run -- k_sgd_tc<64> + k_wgrad_tc<64,64> for
gradients, k_eval_tc<64> for evaluations and predictions, k_gram_dmma +
k_refit for the refit -- on batches of more than 2 x 148 x 2 tiles of 128
rows, so every CTA of the persistent grid walks several tiles (double-buffered
feature prefetch, mbarrier phases across tiles) and the last tile is partial.

Oracle: the FP64 restatement of regressor.cpp (oracle/regress_oracle.c, pinned
by test_oracle_regressor.py).  Tolerances (north star: 1e-5 per path with
identical weights, 1e-3 on trained aggregates):
  * loss 1e-5 relative; every gradient block within 5e-5 of its largest entry;
  * predictions per path: 1e-5 relative + 1e-6 of the largest prediction;
  * refit: the refit network's FP64 loss within 1e-6 of the oracle refit's;
  * train_base at C2 shape: epoch losses and best loss 1e-3, same best epoch.
"""
import json

import numpy as np
import pytest

import cases
import oracle_api
import paper_2211_17005_b200 as hcva
from paper_2211_17005_b200 import regression as rg

pytestmark = pytest.mark.gpu

ACT = {"tanh": 0, "sigmoid": 1, "softplus": 2, "relu": 3}
D, U, H = 45, 64, 2
ROWS = 80_003  # 626 tiles over 296 CTAs: >= 2 tiles per CTA, last tile 3 rows


def tcfg(act="tanh", epochs=8, batches=32, lr=1e-3, adam=True):
    t = hcva.TrainConfig()
    t.width, t.hidden_layers, t.epochs, t.n_batches, t.activation, t.learning_rate, t.adam = (
        U, H, epochs, batches, act, lr, adam)
    return t


def c2_like(rows, seed=1):
    """Standardised C2-like features: 8 default indicators (0/1, passed through
    unscaled) then 37 standardised market columns; a positive label."""
    rng = np.random.default_rng(seed)
    ind = (rng.random((rows, 8)) < np.linspace(0.05, 0.6, 8)).astype(np.float64)
    mk = rng.standard_normal((rows, D - 8))
    x = np.hstack([ind, mk])
    y = np.maximum(0.0, 2.0 + np.sin(mk[:, 0]) + 0.5 * mk[:, 1] * mk[:, 2] - ind[:, :4].sum(1)
                   + 0.3 * rng.standard_normal(rows)) * 10.0
    return x, y


def blocks_close(gg, go, what):
    off = 0
    for fo, fi in [(U, D), (U, U), (1, U)]:
        for blk in (fo * fi, fo):
            a, b = gg[off:off + blk], go[off:off + blk]
            err = np.max(np.abs(a - b))
            assert err <= 5e-5 * max(np.max(np.abs(b)), 1e-12), (what, off, err, np.max(np.abs(b)))
            off += blk
    assert gg[-1] == pytest.approx(go[-1], rel=1e-5, abs=1e-9), what


@pytest.mark.parametrize("act", ["tanh", "sigmoid", "softplus", "relu"])
@pytest.mark.parametrize("head", [False, True])
def test_loss_and_gradients_c2_shape(act, head):
    R = oracle_api.restatement()
    x, y = c2_like(ROWS)
    p = R.init_network(D, H, U, R.key(7, 0xBEEF, 100))
    p[-1] = float(np.mean(y)) * 0.8
    lo, go = R.loss(p, x, y, H, U, ACT[act], head)
    lg, gg = rg.quadratic_loss(tcfg(act), p, x, y, head)
    assert lg == pytest.approx(lo, rel=1e-5)
    blocks_close(gg, go, (act, head))


@pytest.mark.parametrize("act", ["tanh", "relu"])
def test_predictions_per_path_c2_shape(act):
    """k_eval_tc<64>: every one of 80,003 predictions with identical weights."""
    R = oracle_api.restatement()
    x, y = c2_like(ROWS, seed=2)
    p = R.init_network(D, H, U, R.key(7, 0xBEEF, 50))
    p[-1] = float(np.mean(y))
    want = R.forward(p, x, H, U, ACT[act], True)
    got = rg.forward(tcfg(act), p, x)
    err = np.abs(got - want)
    tol = 1e-5 * np.abs(want) + 1e-6 * np.max(np.abs(want))
    assert (err <= tol).all(), f"{(err > tol).sum()} of {err.size} paths, max rel {np.max(err / np.abs(want)):.2e}"


def test_refit_output_layer_c2_shape():
    """k_gram_dmma + k_refit (regressor.cpp:191-213) against the FP64 refit."""
    R = oracle_api.restatement()
    x, y = c2_like(ROWS, seed=3)
    p = R.init_network(D, H, U, R.key(7, 0xBEEF, 10))
    p[-1] = float(np.mean(y))
    want = R.refit(p, x, y, H, U, 1e-8)
    got = rg.refit_output_layer(tcfg(), p, x, y)
    n_out = U + 1  # w_h, b_h just before mu
    assert np.array_equal(got[:-1 - n_out], p[:-1 - n_out]) and got[-1] == p[-1]
    lw = R.loss(want, x, y, H, U, 0, False, grads=False)
    lg = R.loss(got, x, y, H, U, 0, False, grads=False)
    l0 = R.loss(p, x, y, H, U, 0, False, grads=False)
    assert lw < l0
    assert lg == pytest.approx(lw, rel=1e-6)
    wo, wg = want[-1 - n_out:-1], got[-1 - n_out:-1]
    assert np.max(np.abs(wg - wo)) <= 1e-3 * np.max(np.abs(wo))


def test_train_base_c2_shape():
    """One train_base (Alg. 1) on C2-shaped data: 65,536 rows (512 paths x 128
    replicas) in 32 batches of 2048, 8 epochs with the head switch at 4."""
    R = oracle_api.restatement()
    x, y = c2_like(65_536, seed=4)
    t = tcfg()
    init = R.init_network(D, H, U, R.key(7, 0xBEEF, 100))
    init[-1] = float(np.mean(y))
    bo, ro = R.train_base(x, y, init, H, U, t.n_batches, t.epochs, t.learning_rate)
    bg, rgp = rg.train_base(t, x, y, init)
    assert rgp["best_epoch"] == ro["best_epoch"]
    np.testing.assert_allclose(rgp["epoch_losses"], ro["epoch_losses"], rtol=1e-3)
    assert rgp["best_loss"] == pytest.approx(ro["best_loss"], rel=1e-3)
    pg, po = R.forward(bg, x, H, U), R.forward(bo, x, H, U)
    assert np.mean(pg) == pytest.approx(np.mean(po), rel=1e-3)


def test_plain_sgd_train_base():
    """sgd_update (regressor.cpp:236-242): adam = false."""
    R = oracle_api.restatement()
    x, y = c2_like(8192, seed=5)
    t = tcfg(epochs=4, batches=8, lr=1e-4, adam=False)
    init = R.init_network(D, H, U, R.key(3))
    init[-1] = float(np.mean(y))
    bo, ro = R.train_base(x, y, init, H, U, t.n_batches, t.epochs, t.learning_rate, adam=False)
    bg, rgp = rg.train_base(t, x, y, init)
    assert rgp["best_epoch"] == ro["best_epoch"]
    np.testing.assert_allclose(rgp["epoch_losses"], ro["epoch_losses"], rtol=1e-3)
    # plain SGD and Adam move differently from the same start
    ba, _ = rg.train_base(tcfg(epochs=4, batches=8, lr=1e-4, adam=True), x, y, init)
    assert not np.allclose(ba, bg)


def test_divergence_is_numeric_error():
    """regressor.cpp:291-293,319-320: a non-finite loss raises numeric_error."""
    x, y = c2_like(4096, seed=6)
    init = oracle_api.restatement().init_network(D, H, U, 11)
    with pytest.raises(hcva.NumericError, match="diverged"):
        rg.train_base(tcfg(epochs=2, batches=4, lr=1e30, adam=False), x, y * 1e30, init)
    yn = y.copy()
    yn[17] = np.nan
    with pytest.raises(hcva.NumericError, match="diverged"):
        rg.train_base(tcfg(epochs=2, batches=4), x, yn, init)


@pytest.mark.slow
def test_learned_cva_reduced_c2():
    """Alg. 2 on the C2 model with 10 pricing steps, 512 paths x 128 replicas,
    the production network: the per-step learned CVA (mean out-of-sample
    prediction on a validation set, percentile_table's mean) against the FP64
    oracle's Alg. 2 on the same labels.  Each step is trained from the
    engine's own warm start (as test_backward_learn_matches_oracle), so the
    comparison isolates one train_base per step: 1e-3 per step and on the sum."""
    j = cases.case("c2")
    j["grid"]["pricing_steps"] = 10
    cfg = hcva.parse_config(json.dumps(j))
    t = cfg.training
    assert (t.width, t.hidden_layers, t.n_batches) == (U, H, 32)
    book = hcva.generate_book(cfg)
    root = hcva.RandomStream(cfg.seed)
    sim = hcva.simulate_set(cfg, book, 512, 128, root.split(hcva.K_TRAIN_SIM))
    val = hcva.simulate_set(cfg, book, 4096, 1, root.split(hcva.K_VALIDATION_SIM))
    models = rg.backward_learn(sim, t, "defaults")
    table = rg.percentile_table(models, val)
    R = oracle_api.restatement()
    mk, st, cube = sim.market_arrays(), sim.default_steps(), sim.cube_values()
    vmk, vst = val.market_arrays(), val.default_steps()
    got, want = [], []
    for i in range(cfg.n_steps, 0, -1):
        p, mean, scale, rep = models.get(i)
        x = (R.features(i, mk, st) - mean) / scale
        y = R.defaults_label(i, mk, st, cube, cfg.dt).reshape(-1)
        start = models.get(i + 1)[0] if i < cfg.n_steps else R.init_network(
            x.shape[1], t.hidden_layers, t.width, R.key(cfg.seed, 0xBEEF, i))
        if i == cfg.n_steps:
            start[-1] = float(np.mean(y))
        bo, ro = R.train_base(x, y, start, t.hidden_layers, t.width, t.n_batches, t.epochs, t.learning_rate)
        assert rep["best_loss"] == pytest.approx(ro["best_loss"], rel=1e-3), i
        xv = (R.features(i, vmk, vst) - mean) / scale
        cva_o = float(np.mean(R.forward(bo, xv, t.hidden_layers, t.width)))
        assert table[i]["mean"] == pytest.approx(cva_o, rel=1e-3), i
        got.append(table[i]["mean"])
        want.append(cva_o)
    assert sum(got) == pytest.approx(sum(want), rel=1e-3)
