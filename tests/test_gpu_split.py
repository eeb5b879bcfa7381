"""The layer-0 split regression kernels (csrc/regress_split.cu) against the
FP64 oracle on the label source of simulated sets (labels.cpp:142-167,
regressor.cpp:97-158): the feature rows the oracle builds with features_at
are never materialised on the GPU -- the per-path columns y_k and the default
steps go straight into layer 0.

Cases: the paper case's model (E=10, Cc=8: d=45) with U=64 at N=128 (a tile
is one path), N=16 and N=9 (several paths per tile, a path split across
tiles); whole sets and row ranges that cut tiles.  Same tolerances as the
host-row tests: loss 1e-5, gradient blocks 5e-5 of their largest entry,
predictions 1e-5 per path (+1e-6 of the largest)."""
import json

import numpy as np
import pytest

import cases
import oracle_api
import paper_2211_17005_b200 as hcva
from paper_2211_17005_b200 import regression as rg

pytestmark = pytest.mark.gpu

ACT = {"tanh": 0, "sigmoid": 1, "softplus": 2, "relu": 3}
U, H = 64, 2


def c2_set(M, N, steps=4, seed_split=hcva.K_TRAIN_SIM):
    j = cases.case("c2")
    j["grid"]["pricing_steps"] = steps
    cfg = hcva.parse_config(json.dumps(j))
    book = hcva.generate_book(cfg)
    sim = hcva.simulate_set(cfg, book, M, N, hcva.RandomStream(cfg.seed).split(seed_split))
    return cfg, book, sim


def source(R, cfg, sim, i):
    mk, st, cube = sim.market_arrays(), sim.default_steps(), sim.cube_values()
    x = R.features(i, mk, st)
    y = R.defaults_label(i, mk, st, cube, cfg.dt).reshape(-1)
    mean, scale = R.fit_scaler(x, cfg.n_clients)
    return x, y, mean, scale


def tcfg(act="tanh"):
    t = hcva.TrainConfig()
    t.width, t.hidden_layers, t.activation = U, H, act
    return t


def blocks_close(gg, go, d, what):
    off = 0
    for fo, fi in [(U, d), (U, U), (1, U)]:
        for blk in (fo * fi, fo):
            a, b = gg[off:off + blk], go[off:off + blk]
            err = np.max(np.abs(a - b))
            assert err <= 5e-5 * max(np.max(np.abs(b)), 1e-12), (what, off, err, np.max(np.abs(b)))
            off += blk
    assert gg[-1] == pytest.approx(go[-1], rel=1e-5, abs=1e-9), what


@pytest.mark.parametrize("M,N,rows", [(512, 128, None), (512, 128, (1000, 60_001)), (2048, 16, None),
                                      (3000, 9, (5, 26_990)), (4000, 8, None)])
@pytest.mark.parametrize("act,head", [("tanh", False), ("tanh", True), ("relu", True), ("softplus", False)])
def test_split_loss_and_gradients(M, N, rows, act, head):
    R = oracle_api.restatement()
    cfg, book, sim = c2_set(M, N)
    i = 2
    x, y, mean, scale = source(R, cfg, sim, i)
    d = x.shape[1]
    assert d == 45
    p = R.init_network(d, H, U, R.key(cfg.seed, 0xBEEF, i))
    # mu off the label mean: at mu = mean(y) the mu gradient 2 mean(residual)
    # cancels to ~1e-5 of its terms, below the FP32 resolution of a prediction
    p[-1] = 0.8 * float(np.mean(y))
    b0, b1 = rows or (0, x.shape[0])
    xs = (x - mean) / scale
    lo, go = R.loss(p, xs[b0:b1], y[b0:b1], H, U, ACT[act], head)
    lg, gg = rg.sim_quadratic_loss(sim, tcfg(act), i, p, mean, scale, head, rows=(b0, b1))
    assert lg == pytest.approx(lo, rel=1e-5)
    blocks_close(gg, go, d, (M, N, rows, act, head))


def test_split_kernels_run():
    """The timing probe reports whether the split kernels served the set."""
    cfg, book, sim = c2_set(512, 128)
    assert rg.sgd_timing(sim, cfg.training, 2, steps=3)["split"]
    cfg, book, sim = c2_set(64, 4)
    assert not rg.sgd_timing(sim, cfg.training, 2, steps=3)["split"]


def test_split_predictions_validation_set():
    """k_eval_split on a validation set (N = 1: 128 paths per tile) and on a
    training set (N = 128), per path against the FP64 forward."""
    R = oracle_api.restatement()
    cfg, book, sim = c2_set(256, 128, steps=3)
    t = cfg.training
    t.epochs, t.n_batches = 2, 8
    models = rg.backward_learn(sim, t, "defaults")
    val = hcva.simulate_set(cfg, book, 1000, 1, hcva.RandomStream(cfg.seed).split(hcva.K_VALIDATION_SIM))
    for s, i in ((val, 1), (val, 3), (sim, 2)):
        p, mean, scale, _ = models.get(i)
        x = (R.features(i, s.market_arrays(), s.default_steps()) - mean) / scale
        want = R.forward(p, x, H, U)
        got = models.predict(i, s)
        err = np.abs(got - want)
        assert (err <= 1e-5 * np.abs(want) + 1e-6 * np.max(np.abs(want))).all(), (i, err.max())


@pytest.mark.parametrize("M,N", [(256, 128), (2048, 16)])
def test_split_backward_learn_matches_oracle(M, N):
    """Alg. 2 on the split path (persistent epochs): per step, from the
    engine's own warm start, one train_base against the FP64 oracle's (best
    loss 1e-3), and the engine's scaler equal to the oracle's (1e-12)."""
    R = oracle_api.restatement()
    cfg, book, sim = c2_set(M, N, steps=4)
    t = cfg.training
    t.epochs, t.n_batches = 4, 16
    models = rg.backward_learn(sim, t, "defaults")
    assert rg.sgd_timing(sim, t, 2, steps=2)["split"]
    for i in range(cfg.n_steps, 0, -1):
        x, y, mo, so = source(R, cfg, sim, i)
        p, mean, scale, rep = models.get(i)
        assert np.allclose(mean, mo, rtol=1e-12, atol=1e-15) and np.allclose(scale, so, rtol=1e-12)
        xs = (x - mean) / scale
        start = models.get(i + 1)[0] if i < cfg.n_steps else R.init_network(
            x.shape[1], t.hidden_layers, t.width, R.key(cfg.seed, 0xBEEF, i))
        if i == cfg.n_steps:
            start[-1] = float(np.mean(y))
        bo, ro = R.train_base(xs, y, start, t.hidden_layers, t.width, t.n_batches, t.epochs, t.learning_rate)
        assert rep["best_loss"] == pytest.approx(ro["best_loss"], rel=1e-3), i
        assert rep["best_epoch"] == ro["best_epoch"], i


def test_split_deterministic():
    cfg, book, sim = c2_set(256, 128, steps=2)
    t = cfg.training
    t.epochs, t.n_batches = 2, 8
    a = rg.backward_learn(sim, t)
    b = rg.backward_learn(sim, t)
    for i in (1, 2):
        assert np.array_equal(a.get(i)[0], b.get(i)[0])


@pytest.mark.parametrize("M,N", [(256, 128), (2048, 16)])
def test_persistent_epoch_matches_per_step_launches(M, N):
    """The persistent epoch kernel (optimizer fused behind grid barriers) and
    per-step launches (k_sgd_split + k_adam, HCVA_FUSED_EPOCH=0) train the same
    network: the two reduce the same FP32 partial rows in different fixed
    orders in FP64, so they agree to rounding.  N = 128: per-step path parts
    and 16-column slot blocks; N = 16: tiles of 8 paths, 32-column slots."""
    import os
    import subprocess
    import sys

    script = (
        "import json, sys; sys.path.insert(0, 'tests'); sys.path.insert(0, '.');"
        "import numpy as np, cases, paper_2211_17005_b200 as hcva;"
        "from paper_2211_17005_b200 import regression as rg;"
        "j = cases.case('c2'); j['grid']['pricing_steps'] = 2; cfg = hcva.parse_config(json.dumps(j));"
        "t = cfg.training; t.epochs, t.n_batches = 4, 8;"
        f"sim = hcva.simulate_set(cfg, hcva.generate_book(cfg), {M}, {N}, hcva.RandomStream(cfg.seed).split(1));"
        "m = rg.backward_learn(sim, t);"
        "print(json.dumps([list(m.get(i)[0]) for i in (1, 2)] + [rg.sgd_timing(sim, t, 2, steps=2)['fused_step_ms']]))"
    )
    out = {}
    for f in ("1", "0"):
        env = dict(os.environ, HCVA_FUSED_EPOCH=f)
        r = subprocess.run([sys.executable, "-c", script], capture_output=True, text=True, env=env, timeout=600,
                           cwd=oracle_api.ROOT)
        assert r.returncode == 0, r.stderr[-2000:]
        out[f] = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["1"][2] is not None and out["0"][2] is None  # the fused kernel ran only when enabled
    for i in range(2):
        a, b = np.array(out["1"][i]), np.array(out["0"][i])
        assert np.allclose(a, b, rtol=1e-9, atol=1e-12), np.max(np.abs(a - b))
