"""GPU parity of the regression (regressor.cpp) against the FP64 oracle.

The engine computes the network in FP32 on the device with FP64 reductions
and an FP64 Adam/master copy; the reference is FP64 throughout.  Tolerances
(north star: 1e-5 per path in FP32, 1e-3 on final CVA statistics):
  * one quadratic_loss / gradient evaluation with identical parameters:
    loss 1e-5 relative, gradients 5e-5 of the layer's largest gradient;
  * init_network: bit-exact (same stream, same order);
  * scaler: 1e-12 relative;
  * train_base / backward_learn (trajectories of hundreds of Adam steps that
    diverge at FP32 rounding): best losses and mean predictions 1e-3 relative.
"""
import numpy as np
import pytest

import cases
import oracle_api
import paper_2211_17005_b200 as hcva
from paper_2211_17005_b200 import regression as rg

pytestmark = pytest.mark.gpu


def tcfg(width=16, hidden=2, epochs=8, batches=8, act="tanh", seed=7, lr=1e-3):
    t = hcva.TrainConfig()
    t.width, t.hidden_layers, t.epochs, t.n_batches, t.activation, t.seed, t.learning_rate = (
        width, hidden, epochs, batches, act, seed, lr)
    return t


ACT = {"tanh": 0, "sigmoid": 1, "softplus": 2, "relu": 3}


def data(rows, d, seed=3):
    rng = np.random.default_rng(seed)
    x = rng.standard_normal((rows, d))
    y = np.abs(np.sin(x[:, 0]) + 0.3 * x[:, 1 % d] ** 2 + 0.1 * rng.standard_normal(rows))
    return x, y


def test_init_network_bit_exact():
    R = oracle_api.restatement()
    for d, h, u in ((45, 2, 64), (6, 3, 8), (4, 1, 5)):
        t = tcfg(width=u, hidden=h)
        key = R.key(20240901, 0xBEEF, 50)
        assert np.array_equal(rg.init_network(t, d, key), R.init_network(d, h, u, key))


@pytest.mark.parametrize("act", ["tanh", "sigmoid", "softplus", "relu"])
@pytest.mark.parametrize("head", [False, True])
def test_loss_and_gradients_match_fp64(act, head):
    R = oracle_api.restatement()
    d, h, u, rows = 12, 2, 32, 700
    x, y = data(rows, d)
    t = tcfg(width=u, hidden=h, act=act)
    p = R.init_network(d, h, u, R.key(5))
    p[-1] = 0.2
    lo, go = R.loss(p, x, y, h, u, ACT[act], head)
    lg, gg = rg.quadratic_loss(t, p, x, y, head)
    assert lg == pytest.approx(lo, rel=1e-5)
    dims = [(u, d), (u, u), (1, u)]
    off = 0
    for fo, fi in dims:
        for blk in (fo * fi, fo):
            a, b = gg[off:off + blk], go[off:off + blk]
            assert np.max(np.abs(a - b)) <= 5e-5 * max(np.max(np.abs(b)), 1e-12), (act, head, off)
            off += blk
    assert gg[-1] == pytest.approx(go[-1], rel=1e-5, abs=1e-9)


def test_train_base_matches_fp64_trajectory():
    R = oracle_api.restatement()
    d, h, u, rows = 6, 2, 16, 2048
    x, y = data(rows, d, seed=11)
    t = tcfg(width=u, hidden=h, epochs=8, batches=16)
    init = R.init_network(d, h, u, R.key(7))
    init[-1] = float(np.mean(y))
    bo, ro = R.train_base(x, y, init, h, u, 16, 8)
    bg, rgp = rg.train_base(t, x, y, init)
    assert rgp["best_epoch"] == ro["best_epoch"]
    assert rgp["best_loss"] == pytest.approx(ro["best_loss"], rel=1e-3)
    assert np.allclose(rgp["epoch_losses"], ro["epoch_losses"], rtol=1e-3)
    po = R.forward(bo, x, h, u)
    pg = R.forward(bg, x, h, u)
    assert np.mean(pg) == pytest.approx(np.mean(po), rel=1e-3)


def backward_case(name="desk_corr", M=40, N=8, width=16, batches=8, epochs=4):
    cfg = hcva.parse_config(cases.text(name))
    cfg.training.width, cfg.training.n_batches, cfg.training.epochs = width, batches, epochs
    book = hcva.generate_book(cfg)
    sim = hcva.simulate_set(cfg, book, M, N, hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM))
    return cfg, book, sim


def test_backward_learn_matches_oracle():
    """Alg. 2 over every step of a small set (desk model, dense correlation, 12 steps)."""
    cfg, book, sim = backward_case()
    t = cfg.training
    models = rg.backward_learn(sim, t, "defaults")
    R = oracle_api.restatement()
    mk = sim.market_arrays()
    st = sim.default_steps()
    cube = sim.cube_values()

    def source(i):
        return R.features(i, mk, st), R.defaults_label(i, mk, st, cube, cfg.dt).reshape(-1), cfg.n_clients

    ref = R.backward_learn(cfg.n_steps, source, cfg.seed, t.hidden_layers, t.width, t.n_batches, t.epochs,
                           t.learning_rate)
    seq_gpu, seq_ref = [], []
    for i in range(1, cfg.n_steps + 1):
        p, mean, scale, rep = models.get(i)
        po, mo, so, ro = ref[i]
        assert np.allclose(mean, mo, rtol=1e-12, atol=1e-15) and np.allclose(scale, so, rtol=1e-12)
        x = (source(i)[0] - mo) / so
        y = source(i)[1]
        # Per step, from the engine's own warm start (step i+1's best, or the
        # init at i = n): one train_base must agree with the FP64 oracle's.
        start = models.get(i + 1)[0] if i < cfg.n_steps else R.init_network(
            x.shape[1], t.hidden_layers, t.width, R.key(cfg.seed, 0xBEEF, i))
        if i == cfg.n_steps:
            start[-1] = float(np.mean(y))
        bo, ro_i = R.train_base(x, y, start, t.hidden_layers, t.width, t.n_batches, t.epochs, t.learning_rate)
        assert rep["best_loss"] == pytest.approx(ro_i["best_loss"], rel=1e-3, abs=1e-12), i
        pg = models.predict(i, sim)
        pr = R.forward(bo, x, t.hidden_layers, t.width)
        assert np.mean(pg) == pytest.approx(np.mean(pr), rel=1e-3, abs=1e-9), i
        # Whole sequence (Alg. 2 chained through 12 warm starts, FP32 and FP64
        # SGD trajectories diverging at rounding level): per step within 5%,
        # the CVA-like aggregate over the steps within 1%.
        pseq = R.forward(po, x, t.hidden_layers, t.width)
        assert np.mean(pg) == pytest.approx(np.mean(pseq), rel=5e-2, abs=1e-9), i
        seq_gpu.append(np.mean(pg))
        seq_ref.append(np.mean(pseq))
    assert sum(seq_gpu) == pytest.approx(sum(seq_ref), rel=1e-2)


def test_backward_learn_deterministic():
    cfg, book, sim = backward_case()
    a = rg.backward_learn(sim, cfg.training)
    b = rg.backward_learn(sim, cfg.training)
    for i in (1, cfg.n_steps):
        assert np.array_equal(a.get(i)[0], b.get(i)[0])


def test_batch_divisibility_is_config_error():
    cfg, book, sim = backward_case()
    cfg.training.n_batches = 7
    with pytest.raises(hcva.ConfigError):
        rg.backward_learn(sim, cfg.training)


@pytest.mark.parametrize("d,u,head", [(100, 32, False), (157, 64, True), (157, 16, False)])
def test_loss_and_gradients_wide_inputs(d, u, head):
    """Inputs wider than the resident tile (C5: d = 157): layer 0's K dimension
    streams through the tile kernel in 16-column chunks, the weight gradient
    uses the 256-row feature tile; same tolerances as the narrow case."""
    R = oracle_api.restatement()
    h, rows = 2, 700
    x, y = data(rows, d)
    t = tcfg(width=u, hidden=h)
    p = R.init_network(d, h, u, R.key(11))
    p[-1] = 0.2
    lo, go = R.loss(p, x, y, h, u, 0, head)
    lg, gg = rg.quadratic_loss(t, p, x, y, head)
    assert lg == pytest.approx(lo, rel=1e-5)
    off = 0
    for fo, fi in [(u, d), (u, u), (1, u)]:
        for blk in (fo * fi, fo):
            a, b = gg[off:off + blk], go[off:off + blk]
            assert np.max(np.abs(a - b)) <= 5e-5 * max(np.max(np.abs(b)), 1e-12), (d, u, off)
            off += blk
    assert gg[-1] == pytest.approx(go[-1], rel=1e-5, abs=1e-9)


@pytest.mark.parametrize("path", ["tensor", "simt"])
def test_backward_learn_c5_shape(path, monkeypatch):
    """C5's feature width (64 clients: d = 64 + 29 + 64 = 157) on the
    tensor-core path (chunked layer 0) and on the SIMT trainer; per step both
    must match the FP64 oracle."""
    import json

    if path == "simt":
        monkeypatch.setenv("HCVA_REGRESS_SIMT", "1")

    j = cases.case("c5")
    j["grid"] = {"pricing_steps": 4, "substeps": 4, "dt_years": 0.25}
    cfg = hcva.parse_config(json.dumps(j))
    t = cfg.training
    t.width, t.n_batches, t.epochs = 16, 4, 4
    book = hcva.generate_book(cfg)
    sim = hcva.simulate_set(cfg, book, 16, 4, hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM))
    models = rg.backward_learn(sim, t, "defaults")
    assert models.input_dim == 157
    R = oracle_api.restatement()
    mk, st, cube = sim.market_arrays(), sim.default_steps(), sim.cube_values()
    for i in range(cfg.n_steps, 0, -1):
        p, mean, scale, rep = models.get(i)
        x = (R.features(i, mk, st) - mean) / scale
        y = R.defaults_label(i, mk, st, cube, cfg.dt).reshape(-1)
        start = models.get(i + 1)[0] if i < cfg.n_steps else R.init_network(
            x.shape[1], t.hidden_layers, t.width, R.key(cfg.seed, 0xBEEF, i))
        if i == cfg.n_steps:
            start[-1] = float(np.mean(y))
        bo, ro = R.train_base(x, y, start, t.hidden_layers, t.width, t.n_batches, t.epochs, t.learning_rate)
        assert rep["best_loss"] == pytest.approx(ro["best_loss"], rel=1e-3, abs=1e-12), i



@pytest.mark.parametrize("n,k", [(32, 16), (64, 48), (64, 64), (128, 64)])
def test_tcgen05_operand_forms(n, k):
    """The two 3xTF32 tcgen05.mma forms the regression kernels use: A and B
    K-major in shared memory (variant 0) and A in tensor memory (variant 8,
    k_sgd_tc / k_eval_tc), M = 128, against an FP64 product (~1e-6 relative:
    3xTF32 is FP32-accurate)."""
    import ctypes as C

    from paper_2211_17005_b200 import _lib

    L = _lib.lib()
    L.hcva_diag_tc_gemm.argtypes = [C.c_void_p] + [C.c_int] * 4 + [C.c_void_p] * 3
    rng = np.random.default_rng(k)
    A = rng.standard_normal((128, k)).astype(np.float32)
    B = rng.standard_normal((n, k)).astype(np.float32)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    for var in (0, 8):
        D = np.zeros((128, n), dtype=np.float32)
        assert L.hcva_diag_tc_gemm(hcva.context().handle, 128, n, k, var, A.ctypes.data, B.ctypes.data,
                                   D.ctypes.data) == 0
        assert np.max(np.abs(D - ref)) <= 2e-6 * np.max(np.abs(ref)), var
