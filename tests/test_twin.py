"""Twin-MC validator: twin_labels on the GPU against the
golden labels and, at larger sizes, the restatement.  The estimators of
validation.cpp:41-117 are tested in test_estimators.py."""
import numpy as np
import pytest

import cases
import oracle_api
import paper_2211_17005_b200 as hcva

GOLDEN = ["minimal", "c1", "desk_corr", "c2", "c5"]


def golden(name):
    return np.load(f"{oracle_api.ROOT}/tests/golden/{name}.npz")


def gpu_twin(name, M, N, step):
    cfg = hcva.parse_config(cases.text(name))
    book = hcva.generate_book(cfg)
    sim = hcva.simulate_set(cfg, book, M, N, hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM))
    t1, t2 = hcva.twin_labels(sim, book, step, hcva.RandomStream(cfg.seed).split(2).split(4).split(step))
    return cfg, book, sim, t1, t2


def close(got, want, rtol, what):
    scale = np.max(np.abs(want)) if want.size else 0.0
    bad = np.abs(got - want) > rtol * np.abs(want) + 1e-12 * scale + 1e-300
    assert not bad.any(), f"{what}: {bad.sum()} / {bad.size} labels outside tolerance"


@pytest.mark.gpu
@pytest.mark.parametrize("name", GOLDEN)
def test_twin_labels_vs_golden(name):
    z = golden(name)
    _, _, _, t1, t2 = gpu_twin(name, int(z["M"]), int(z["N"]), int(z["twin_step"]))
    # continuation market 1e-11, cube 1e-10 of scale: labels 1e-9; a re-sampled
    # default landing on a different step would miss by a whole term.
    close(t1, z["twin1"], 1e-9, "twin1")
    close(t2, z["twin2"], 1e-9, "twin2")
    assert (t1 > 0).any() and not np.array_equal(t1, t2)


@pytest.mark.gpu
@pytest.mark.parametrize("name,M,N,step", [("c1", 384, 16, 0), ("c1", 384, 16, 49), ("desk_corr", 200, 8, 11),
                                           ("c1", 64, 4, 50)])
def test_twin_labels_vs_restatement(name, M, N, step):
    cfg, book, sim, t1, t2 = gpu_twin(name, M, N, step)
    R = oracle_api.restatement()
    m = cases.oracle_model(cfg)
    r1, r2 = R.twin_labels(m, book, step, sim.market_arrays(), sim.default_steps(),
                           R.key(cfg.seed, 2, 4, step))
    close(t1, r1, 1e-9, "twin1")
    close(t2, r2, 1e-9, "twin2")
    if step == cfg.n_steps:
        assert not t1.any() and not t2.any()


@pytest.mark.gpu
def test_twin_label_mean_matches_defaults_label_mean():
    """Each twin is a fresh draw of the same conditional law as the pathwise
    defaults label (labels.cpp:21-48 vs :90-140): their sample means agree
    statistically at a large size."""
    cfg, book, sim, t1, t2 = gpu_twin("c1", 4096, 16, 10)
    lab = sim.labels(10, "defaults")
    se = np.std(lab) / np.sqrt(lab.size)
    assert abs(np.mean(t1) - np.mean(lab)) < 6 * se and abs(np.mean(t2) - np.mean(lab)) < 6 * se
