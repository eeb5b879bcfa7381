"""ARD variance sampling (ard.cpp:56-125) on the GPU
against the FP64 restatement (whose parts -- market, defaults, cube, labels --
are pinned bit-exact to the compiled reference; the reference's ard.cpp itself
needs Eigen).  Default indicators are bit-exact, so v_x is compared exactly."""
import numpy as np
import pytest

import cases
import oracle_api
import paper_2211_17005_b200 as hcva

PRIOR = [0.5, 1.5, 0.5, 2.0, 0.5, 1.5]


def test_restated_ard_shapes_and_positivity():
    cfg = hcva.parse_config(cases.text("desk_corr"))
    R = oracle_api.restatement()
    m = cases.oracle_model(cfg)
    book = R.generate_book(m, 12, 1.0, 25.0, R.key(cfg.seed, 0))
    out = R.ard_sample_variances(m, book, PRIOR, 3, 24, R.key(cfg.seed, 9))
    assert out["v_x"].shape == (3, cfg.n_clients) and out["v_y"].shape == (3, 2 * cfg.n_economies - 1 + cfg.n_clients)
    assert np.all(out["v_y"] >= 0) and np.all(out["v_x"] >= 0) and np.all(out["v_xi"] > 0)
    assert out["rejected"] == 0
    # different draws move the variances
    assert not np.allclose(out["v_y"][0], out["v_y"][1])


@pytest.mark.gpu
@pytest.mark.parametrize("name,n_dgp,paths", [("desk_corr", 4, 48), ("c1", 3, 64)])
def test_ard_vs_restatement(name, n_dgp, paths):
    cfg = hcva.parse_config(cases.text(name))
    book = hcva.generate_book(cfg)
    stream = hcva.RandomStream(cfg.seed).split(9)
    got = hcva.ard_sample_variances(cfg, book, n_dgp, paths, stream)
    R = oracle_api.restatement()
    want = R.ard_sample_variances(cases.oracle_model(cfg), book, PRIOR, n_dgp, paths, stream.key)
    assert got["rejected"] == want["rejected"]
    assert np.array_equal(got["v_x"], want["v_x"])
    for k in ("v_y", "v_xi"):
        assert np.allclose(got[k], want[k], rtol=1e-9, atol=0), k
