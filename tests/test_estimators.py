"""Validation statistics reduced on the GPU (csrc/estimators.cu) against the
compiled reference (oracle/_ref: validation.cpp:41-117,181-210,
planner.cpp:11-70), the golden fixtures it produced, and the restatement
(percentile_table, pipeline.cpp:41-47,138-156, whose source needs Eigen).

The device reductions sum in a fixed tree order, the reference sequentially,
so the bar is rounding level: 1e-12 relative (plus 1e-15 of the data scale
for values that cancel to ~0), and exact equality of the counts."""
import numpy as np
import pytest

import cases
import oracle_api
import paper_2211_17005_b200 as hcva
from paper_2211_17005_b200 import regression as rg

GOLDEN = ["minimal", "c1", "desk_corr", "c2", "c5"]
RTOL = 1e-12


def checker():
    """The compiled reference where it was built, else the pinned restatement."""
    return oracle_api.reference() or oracle_api.restatement()


def near(got, want, scale=0.0):
    got, want = np.asarray(got, dtype=float), np.asarray(want, dtype=float)
    ok = np.abs(got - want) <= RTOL * np.abs(want) + 1e-15 * scale
    return bool(np.all(ok | (np.isnan(got) & np.isnan(want))))


def estimators(t1, t2, N):
    pred = cases.twin_prediction(t1, t2)
    out = []
    for block in (1, N):
        out += list(hcva.twin_l2_error(pred, t1, t2, block))
    try:
        out.append(hcva.twin_relative_rmse(pred, t1, t2))
    except hcva.NumericError:
        out.append(float("nan"))
    out += [hcva.twin_relative_rmse_std_error(pred, t1, t2, b) for b in (1, N)]
    return np.array(out)


@pytest.mark.gpu
@pytest.mark.parametrize("name", GOLDEN)
def test_twin_estimators_vs_golden(name):
    z = np.load(f"{oracle_api.ROOT}/tests/golden/{name}.npz")
    t1, t2 = z["twin1"], z["twin2"]
    scale = float(np.max(np.abs(t1 * t2))) if t1.size else 0.0
    assert near(estimators(t1, t2, int(z["N"])), z["twin_stats"], scale)


@pytest.mark.gpu
@pytest.mark.parametrize("n,block", [(1000, 8), (97, 1), (64, 64), (2, 1), (4096 * 16, 16), (33 * 128, 128),
                                     (100, 7)])
def test_twin_estimators_random(n, block):
    F = checker()
    rng = np.random.default_rng(n + block)
    t1 = rng.exponential(size=n) * (rng.random(n) < 0.6)
    t2 = rng.exponential(size=n) * (rng.random(n) < 0.6)
    pred = rng.random(n)
    assert near(hcva.twin_l2_error(pred, t1, t2, block), F.twin_l2_error(pred, t1, t2, block), 1.0)
    if np.mean(t1 * t2) > 0:
        assert near(hcva.twin_relative_rmse(pred, t1, t2), F.twin_relative_rmse(pred, t1, t2))
    else:
        with pytest.raises(hcva.NumericError):
            hcva.twin_relative_rmse(pred, t1, t2)
    assert near(hcva.twin_relative_rmse_std_error(pred, t1, t2, block),
                F.twin_relative_rmse_std_error(pred, t1, t2, block))


@pytest.mark.gpu
def test_twin_estimator_errors():
    with pytest.raises(hcva.ContractError):
        hcva.twin_l2_error(np.zeros(3), np.zeros(3), np.zeros(2))
    with pytest.raises(hcva.NumericError):
        hcva.twin_relative_rmse(np.ones(4), np.zeros(4), np.ones(4))


@pytest.mark.gpu
@pytest.mark.parametrize("n", [2, 3, 39, 40, 41, 1000, 4096, 16384])
def test_estimate_qr(n):
    F = checker()
    rng = np.random.default_rng(n)
    g1 = rng.gamma(2.0, 1.0, n)
    g2 = 0.6 * g1 + rng.gamma(2.0, 0.5, n)
    got, want = rg.estimate_qr(g1, g2), F.estimate_qr(g1, g2)
    assert got["n_pairs"] == want["n_pairs"] == n
    for k in ("q", "r", "total", "q_std_error", "r_std_error"):
        assert near(got[k], want[k], want["total"]), (k, got[k], want[k])


@pytest.mark.gpu
def test_estimate_qr_errors():
    with pytest.raises(hcva.NumericError):
        rg.estimate_qr([1.0], [2.0])
    with pytest.raises(hcva.ContractError):
        rg.estimate_qr([1.0, 2.0], [2.0])


@pytest.mark.gpu
@pytest.mark.parametrize("n,zeros", [(1, 0), (2, 0), (16384, 0), (5000, 700), (3, 2)])
def test_nested_relative_rmse(n, zeros):
    F = checker()
    rng = np.random.default_rng(n + zeros)
    nested = rng.gamma(2.0, 0.01, n)
    nested[rng.permutation(n)[:zeros]] = 0.0
    pred = nested * (1.0 + 0.1 * rng.standard_normal(n)) + 1e-4 * rng.random(n)
    got, want = hcva.nested_relative_rmse(pred, nested), F.nested_relative_rmse(pred, nested)
    assert got[2:] == want[2:]
    assert near(got[:2], want[:2])


@pytest.mark.gpu
def test_nested_relative_rmse_errors():
    with pytest.raises(hcva.NumericError):
        hcva.nested_relative_rmse(np.ones(3), np.zeros(3))
    with pytest.raises(hcva.ContractError):
        hcva.nested_relative_rmse(np.ones(3), np.ones(2))
    with pytest.raises(hcva.ContractError):
        hcva.nested_relative_rmse(np.ones(0), np.ones(0))


def test_nested_relative_rmse_restatement_pinned_to_reference():
    F = oracle_api.reference()
    if F is None:
        pytest.skip("compiled reference not built here (no /root/reference)")
    R = oracle_api.restatement()
    rng = np.random.default_rng(3)
    for n, zeros in ((1, 0), (7, 3), (1000, 10)):
        nested = rng.gamma(2.0, 0.01, n)
        nested[:zeros] = 0.0
        pred = nested + 1e-3 * rng.random(n)
        assert R.nested_relative_rmse(pred, nested) == F.nested_relative_rmse(pred, nested)


def test_percentile_restatement_interpolation():
    """percentile_sorted (pipeline.cpp:41-47) by hand on small sorted arrays."""
    R = oracle_api.restatement()
    v = np.arange(101, dtype=float)  # pos = q * 100
    np.testing.assert_array_equal(R.percentile_bands(v[::-1]), [50.0, 1.0, 2.5, 97.5, 99.0])
    np.testing.assert_array_equal(R.percentile_bands(np.array([3.0])), [3.0, 3.0, 3.0, 3.0, 3.0])
    np.testing.assert_allclose(R.percentile_bands(np.array([2.0, 0.0])), [1.0, 0.02, 0.05, 1.95, 1.98])


@pytest.mark.gpu
def test_percentile_table_vs_restatement():
    """percentile_table (pipeline.cpp:138-156) on a trained sequence: the GPU's
    bands equal the restatement's on the engine's own predictions."""
    cfg = hcva.parse_config(cases.text("desk_corr"))
    cfg.n_steps = 6
    cfg.training.width, cfg.training.n_batches, cfg.training.epochs = 16, 4, 4
    book = hcva.generate_book(cfg)
    root = hcva.RandomStream(cfg.seed)
    sim = hcva.simulate_set(cfg, book, 64, 8, root.split(hcva.K_TRAIN_SIM))
    models = rg.backward_learn(sim, cfg.training)
    val = hcva.simulate_set(cfg, book, 333, 1, root.split(2))
    table = rg.percentile_table(models, val)
    R = oracle_api.restatement()
    assert sorted(table) == list(range(1, cfg.n_steps + 1))
    for i, row in table.items():
        pred = models.predict(i, val)
        want = R.percentile_bands(pred)
        got = [row[k] for k in ("mean", "p1", "p2_5", "p97_5", "p99")]
        assert near(got, want, float(np.max(np.abs(pred)))), (i, got, want)
