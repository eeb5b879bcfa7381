"""Q/R probe: estimate_qr (planner.cpp:11-70) on the
GPU (test_estimators.py) against the compiled reference and the restatement; the
probe's default block / labels on the GPU against the oracle; the per-epoch
(Q, R) trace of backward_learn checked at each step's best epoch against the
FP64 forward of the trained network on the probe rows."""
import numpy as np
import pytest

import cases
import oracle_api
import paper_2211_17005_b200 as hcva
from paper_2211_17005_b200 import regression as rg


def _pairs(rng, n):
    g1 = rng.gamma(2.0, 1.0, n)
    return g1, 0.6 * g1 + rng.gamma(2.0, 0.5, n)


def test_estimate_qr_restatement_pinned_to_reference():
    F = oracle_api.reference()
    if F is None:
        pytest.skip("compiled reference not built here (no /root/reference)")
    R = oracle_api.restatement()
    rng = np.random.default_rng(10)
    for n in (2, 7, 40, 333):
        g1, g2 = _pairs(rng, n)
        assert R.estimate_qr(g1, g2) == F.estimate_qr(g1, g2)
        q = F.estimate_qr(g1, g2)
        assert q["q"] + q["r"] == pytest.approx(q["total"], rel=1e-12)


def _case(name="desk_corr", M=64, N=8, width=16, batches=8, epochs=4):
    cfg = hcva.parse_config(cases.text(name))
    cfg.training.width, cfg.training.n_batches, cfg.training.epochs = width, batches, epochs
    book = hcva.generate_book(cfg)
    root = hcva.RandomStream(cfg.seed)
    sim = hcva.simulate_set(cfg, book, M, N, root.split(hcva.K_TRAIN_SIM))
    return cfg, book, sim, root.split(hcva.K_TRAIN_SIM).split(2)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["defaults", "intensity"])
def test_probe_block_vs_oracle(kind):
    cfg, book, sim, probe = _case()
    R = oracle_api.restatement()
    st, lab = rg.probe_block(sim, probe, kind)
    mk = sim.market_arrays()
    ref_st = R.sample_defaults(mk["hazard"], 2, probe.key)
    assert np.array_equal(st, ref_st)
    fn = R.defaults_label if kind == "defaults" else R.intensity_label
    cube = sim.cube_values()
    for i in (0, 3, cfg.n_steps):
        want = fn(i, mk, ref_st, cube, cfg.dt)
        err = np.abs(lab[i] - want)
        assert np.all(err <= 1e-9 * np.abs(want) + 1e-12 * max(np.max(np.abs(want)), 1e-300)), i


@pytest.mark.gpu
def test_qr_trace_at_best_epoch_matches_fp64_forward():
    cfg, book, sim, probe = _case()
    t = cfg.training
    plain = rg.backward_learn(sim, t, "defaults")
    models = rg.backward_learn(sim, t, "defaults", qr_probe=probe)
    tr = models.qr_trace
    n, E = cfg.n_steps, t.epochs
    assert tr.shape == (n * E, 4)
    assert np.array_equal(tr[:, 0], np.repeat(np.arange(n, 0, -1), E))
    assert np.array_equal(tr[:, 1], np.tile(np.arange(1, E + 1), n))
    R = oracle_api.restatement()
    mk = sim.market_arrays()
    st, lab = rg.probe_block(sim, probe, "defaults")
    M = sim.n_paths
    for i in range(1, n + 1):
        p, mean, scale, rep = models.get(i)
        assert np.array_equal(p, plain.get(i)[0]), i  # the probe does not perturb training
        x = (R.features(i, mk, st) - mean) / scale
        pred = R.forward(p, x, t.hidden_layers, t.width).reshape(M, 2)
        g = (pred - lab[i]) ** 2
        qr = R.estimate_qr(g[:, 0], g[:, 1])
        row = tr[(n - i) * E + rep["best_epoch"] - 1]
        tol = 1e-4 * qr["total"] + 1e-300
        assert abs(row[2] - qr["q"]) <= tol and abs(row[3] - qr["r"]) <= tol, (i, row, qr)
