"""The reference's analytic test cases, run on the GPU engine (the oracle pins
the same cases in test_oracle_pin.py): zero-volatility replay
(test_market.cpp:95-118), par swaps worth zero at inception
(test_portfolio.cpp:85-105), and nested CVA against its deterministic closed
form (test_validation.cpp:108-135)."""
import json
import math

import numpy as np
import pytest

import paper_2211_17005_b200 as hcva

pytestmark = pytest.mark.gpu


def config(economies, bank, clients, steps, substeps, dt=1.0, seed=5, swaps=3):
    j = {
        "seed": seed,
        "model": {"economies": [dict(zip(("a", "b", "sigma", "r0"), e)) for e in economies],
                  "bank": dict(zip(("alpha", "delta", "nu", "gamma0"), bank)),
                  "clients": [dict(zip(("alpha", "delta", "nu", "gamma0"), c)) for c in clients]},
        "grid": {"pricing_steps": steps, "substeps": substeps, "dt_years": dt},
        "book": {"generate": {"count": swaps, "notional_min": 1.0, "notional_max": 10.0}},
        "simulation": {"paths": 4, "replicas": 2},
    }
    return hcva.parse_config(json.dumps(j))


def test_zero_vol_replay():
    """Zero vols: every path follows the deterministic Euler scheme (1e-13)."""
    cfg = config([(0.5, 0.03, 0.0, 0.02)], (0.3, 0.01, 0.0, 0.01), [(0.5, 0.02, 0.0, 0.015)], 4, 8)
    sim = hcva.simulate_set(cfg, hcva.generate_book(cfg), 3, 2, hcva.RandomStream(5))
    mk = sim.market_arrays()
    h = 1.0 / 8
    r, g1, lb, lam = 0.02, 0.015, 0.0, 0.0
    for i in range(1, 5):
        for _ in range(8):
            lb += r * h
            lam += g1 * h
            r += 0.5 * (0.03 - r) * h
            g1 += 0.5 * (0.02 - g1) * h
        for k in range(3):
            assert mk["rates"][k, i, 0] == pytest.approx(r, rel=1e-13)
            assert mk["disc"][k, i] == pytest.approx(math.exp(-lb), rel=1e-13)
            assert mk["hazard"][k, i, 1] == pytest.approx(lam, rel=1e-13)


@pytest.mark.parametrize("mat", [1, 4, 10])
def test_par_swap_prices_zero(mat):
    """A swap at its par rate is worth zero at t = 0 on every path; past its
    maturity it drops out of the cube."""
    v = (0.5, 0.03, 0.01, 0.02)
    cfg = config([v], (0.3, 0.01, 0.05, 0.01), [(0.5, 0.05, 0.1, 0.04)], 10, 1)
    rate = hcva.par_rate(float(mat), 1.0, cfg.rates[0])
    book = np.zeros(1, dtype=hcva.generate_book(cfg).dtype)
    book[0] = (0, 1, 1.0, 1.0, float(mat), rate)
    cube = hcva.simulate_set(cfg, book, 8, 2, hcva.RandomStream(1)).cube_values()
    assert np.all(np.abs(cube[:, 0, 0]) < 1e-12)
    assert np.all(cube[:, mat + 1:, 0] == 0.0)


def test_nested_cva_matches_closed_form_at_zero_vols():
    """Deterministic market and constant hazard: the nested estimate is
    sum_{j=i}^{n-1} beta_i^-1 beta_j (MtM_j)^+ gamma dt exp(-gamma (j-i) dt),
    with zero standard error."""
    gamma = 0.03
    cfg = config([(0.5, 0.03, 0.0, 0.02)], (0.3, 0.01, 0.0, 0.01), [(0.0, 0.05, 0.0, gamma)], 8, 8)
    book = hcva.generate_book(cfg)
    sim = hcva.simulate_set(cfg, book, 1, 1, hcva.RandomStream(5))
    mk, cube = sim.market_arrays(), sim.cube_values()
    i, n = 2, 8
    st = {k: v[None, :] for k, v in sim.state_at(0, i).items()}
    val, se = hcva.nested_cva(cfg, book, st, np.array([[True]]), i, 16, hcva.RandomStream(5).split(2))
    want = sum(mk["disc"][0, j] / mk["disc"][0, i] * max(cube[0, j, 0], 0.0) * gamma * cfg.dt *
               math.exp(-gamma * (j - i) * cfg.dt) for j in range(i, n))
    assert want > 0.0
    assert val[0] == pytest.approx(want, rel=1e-8)
    assert se[0] < 1e-12
