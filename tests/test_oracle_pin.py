"""Pin the CPU oracle (oracle/hcva_oracle.c) before trusting it as the checker.

1. SURVEY.md 8c known-answer draws of the compiled reference.
2. The committed golden fixtures (tests/golden/*.npz, produced by the compiled
   reference via tests/golden/make_golden.py): bit-identical.
3. Live comparison against oracle/_ref (the reference's own sources) where
   it was built: bit-identical on fresh configs.
4. The reference's own analytic tests, restated (test_market.cpp:95-118,
   test_defaults.cpp:26-36, test_portfolio.cpp:85-105).
"""
import json
import math

import numpy as np
import pytest

import cases
import oracle_api
from paper_2211_17005_b200.config import parse_config

GOLDEN = ["minimal", "c1", "desk_corr", "c2", "c5"]


@pytest.fixture(scope="module")
def R():
    return oracle_api.restatement()


def test_survey_kats(R):
    k = R.key(42)
    assert [int(x) for x in R.u64(k, 0, 4)] == [
        0xCA8C049A4F3149C9, 0x440A2B7924D0B448, 0x403AB8683F161892, 0xE5BB754197A404D7]
    # SURVEY.md's line evaluated next_uniform/next_normal/next_exponential as
    # printf arguments (right-to-left on x86-64 gcc): uniform = draw 2,
    # normal = draw 1, exponential = draw 0.
    assert R.uniforms(k, 2, 1)[0] == 0.25089600129202733
    assert R.normals(k, 1, 1)[0] == -0.6256258822715044
    assert R.exponentials(k, 0, 1)[0] == 0.23420575649131969
    assert R.normals(R.key(7, 1, 0, 3), 0, 1)[0] == 0.53603967906048189


def test_rng_golden(R):
    z = np.load(oracle_api.ROOT + "/tests/golden/rng_kat.npz")
    k42 = R.key(42)
    assert int(z["keys"][0]) == k42 and int(z["keys"][3]) == R.key(7, 1, 0, 3)
    assert int(z["keys"][1]) == R.split(k42, 0) and int(z["keys"][2]) == R.split(k42, 1)
    assert np.array_equal(R.u64(k42, 0, 64), z["u64_42"])
    assert np.array_equal(R.uniforms(k42, 0, 64), z["uniform_42"])
    assert np.array_equal(R.normals(k42, 0, 4096), z["normal_42"])
    assert np.array_equal(R.exponentials(k42, 0, 256), z["exp_42"])
    assert np.array_equal(R.normals(R.key(7, 1, 0, 3), 0, 256), z["normal_7_1_0_3"])


def run_case(O, name, M, N, steps, fstep, nested, tstep=None):
    cfg = parse_config(cases.text(name))
    m = cases.oracle_model(cfg)
    root = O.key(cfg.seed)
    book = O.generate_book(m, cfg.book_count, cfg.notional_min, cfg.notional_max, O.split(root, 0))
    sk = O.split(root, 1)
    mk = O.simulate_market(m, M, O.split(sk, 0))
    st = O.sample_defaults(mk["hazard"], N, O.split(sk, 1))
    cube = O.build_cube(m, mk, book)
    out = dict(book=book, steps=st, cube=cube)
    for k, v in mk.items():
        out["market_" + k] = v
    out["labels_defaults"] = np.stack([O.defaults_label(i, mk, st, cube, cfg.dt) for i in steps])
    out["labels_intensity"] = np.stack([O.intensity_label(i, mk, st, cube, cfg.dt) for i in steps])
    out["features"] = O.features(fstep, mk, st)
    step, states, inner = nested
    vals = []
    for s in range(states):
        state = dict(rates=mk["rates"][s, step], log_fx=np.log(mk["fx"][s, step]),
                     intens=mk["intens"][s, step], lagged=mk["lagged"][s, step])
        surv = (st[s, 0, 1:] > step).astype(np.int32)
        vals.append(O.nested_cva(m, book, state, surv, step, inner, O.key(cfg.seed, 2, 3, step, s)))
    out["nested"] = np.array(vals)
    if tstep is not None:
        out["twin1"], out["twin2"], out["twin_stats"] = cases.twin_block(O, cfg, m, book, mk, st, tstep)
    return out


@pytest.mark.parametrize("name", GOLDEN)
def test_restatement_matches_golden_bit_exact(R, name):
    z = np.load(f"{oracle_api.ROOT}/tests/golden/{name}.npz")
    got = run_case(R, name, int(z["M"]), int(z["N"]), list(z["label_steps"]), int(z["feature_step"]),
                   tuple(int(x) for x in z["nested_spec"]), int(z["twin_step"]))
    for key, v in got.items():
        assert np.array_equal(v, z[key], equal_nan=key == "twin_stats"), key


def test_restatement_matches_compiled_reference_live(R):
    F = oracle_api.reference()
    if F is None:
        pytest.skip("compiled reference not built here (no /root/reference)")
    # A configuration not among the fixtures: 2 economies, 3 clients, odd D.
    j = cases.case("desk_corr")
    j["model"].pop("brownian_correlation")
    j["model"]["economies"] = j["model"]["economies"][:2]
    j["model"]["clients"] = j["model"]["clients"][:3]
    j["seed"] = 99
    j["grid"] = {"pricing_steps": 7, "substeps": 3, "dt_years": 0.75}
    cfg = parse_config(json.dumps(j))
    m = cases.oracle_model(cfg)
    outs = []
    for O in (R, F):
        root = O.key(cfg.seed)
        book = O.generate_book(m, 15, 1.0, 50.0, O.split(root, 0))
        mk = O.simulate_market(m, 33, O.split(O.split(root, 1), 0))
        st = O.sample_defaults(mk["hazard"], 5, O.split(O.split(root, 1), 1))
        cube = O.build_cube(m, mk, book)
        lab = [O.defaults_label(i, mk, st, cube, cfg.dt) for i in range(cfg.n_steps + 1)]
        il = [O.intensity_label(i, mk, st, cube, cfg.dt) for i in range(cfg.n_steps + 1)]
        state = dict(rates=mk["rates"][3, 2], log_fx=np.log(mk["fx"][3, 2]), intens=mk["intens"][3, 2],
                     lagged=mk["lagged"][3, 2])
        cond = O.simulate_conditional(m, state, 2, 4, 9, O.key(5, 1))
        twin = cases.twin_block(O, cfg, m, book, mk, st, 3)
        outs.append([book, mk, st, cube, lab, il, cond, twin])
    a, b = outs
    assert np.array_equal(a[0], b[0])
    for k in a[1]:
        assert np.array_equal(a[1][k], b[1][k]), k
    assert np.array_equal(a[2], b[2]) and np.array_equal(a[3], b[3])
    assert all(np.array_equal(x, y) for x, y in zip(a[4], b[4]))
    assert all(np.array_equal(x, y) for x, y in zip(a[5], b[5]))
    for k in a[6]:
        assert np.array_equal(a[6][k], b[6][k]), k
    assert all(np.array_equal(x, y, equal_nan=True) for x, y in zip(a[7], b[7]))


def small_model(**kw):
    m = dict(rates=[[0.5, 0.03, 0.01, 0.02]], fx=np.zeros((0, 3)),
             credit=[[0.3, 0.01, 0.05, 0.01], [0.5, 0.02, 0.08, 0.015]], corr=None,
             n_steps=4, substeps=8, dt=1.0)
    m.update(kw)
    return m


def test_zero_vol_replay(R):
    """test_market.cpp:95-118: zero vols reduce to the deterministic scheme (1e-13)."""
    m = small_model(rates=[[0.5, 0.03, 0.0, 0.02]], credit=[[0.3, 0.01, 0.0, 0.01], [0.5, 0.02, 0.0, 0.015]])
    mk = R.simulate_market(m, 3, R.key(5))
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


def test_default_step_arithmetic(R):
    """test_defaults.cpp:26-36 restated through sample_defaults: thresholds are
    compared with >= against pricing-step hazards (ties count as default)."""
    key = R.key(3)
    eps = R.exponentials(R.split(R.split(key, 0), 0), 0, 2)  # names 0 and 1 of replica (0,0)
    n = 10
    lam = np.zeros((1, n + 1, 2))
    lam[0, :, 0] = np.linspace(0, 0.02 * n, n + 1) * 0.0 + eps[0]  # every step ties exactly
    lam[0, :, 1] = np.arange(n + 1) * (eps[1] / 3.0)
    lam[0, 3, 1] = eps[1]  # exact tie at step 3
    st = R.sample_defaults(lam, 1, key)
    assert st[0, 0, 0] == 0
    assert st[0, 0, 1] == 3
    lam[0, :, 1] = np.minimum(lam[0, :, 1], eps[1] * 0.999)
    st = R.sample_defaults(lam, 1, key)
    assert st[0, 0, 1] == 0xFFFF


def test_par_swap_prices_zero(R):
    """test_portfolio.cpp:85-105: a par swap is worth 0 at t = 0 (1e-12)."""
    m = small_model(n_steps=10, substeps=1)
    v = [0.5, 0.03, 0.01, 0.02]
    for mat in (1, 4, 10):
        rate = R.par_rate(float(mat), 1.0, v)
        book = np.array([(0, 1, 1.0, 1.0, float(mat), rate)], dtype=oracle_api.SWAP_DTYPE)
        mk = R.simulate_market(m, 2, R.key(1))
        cube = R.build_cube(m, mk, book)
        assert abs(cube[0, 0, 0]) < 1e-12
        assert np.all(cube[:, mat + 1:, 0] == 0.0)  # expired swaps drop out
