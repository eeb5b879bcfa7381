"""Shared parity cases (reference JSON schema, proj/src/config.cpp:46-172).

C1 / C2 follow SURVEY.md section 8d: C1 = economy 0 and clients 1-2 of
configs/desk.json with the desk bank, 10 swaps, n=50, sub=25; C2 =
configs/paper_shape.json with quarterly steps.
"""
import copy
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _load(name):
    with open(os.path.join(ROOT, "configs", name)) as f:
        return json.load(f)


def _desk_corr():
    """A dense PSD Brownian correlation for the desk model (D = 2*3-1+5 = 10),
    with the pinned (r_e, chi_e) entries equal to rho_e (market.cpp:39-46)."""
    d = 10
    rng = np.random.default_rng(123)
    a = rng.standard_normal((d, 3 * d))
    c = a @ a.T
    s = np.sqrt(np.diag(c))
    c = c / np.outer(s, s) * 0.35
    np.fill_diagonal(c, 1.0)
    c[1, 3] = c[3, 1] = -0.25   # (r_1, chi_1) = rho_1
    c[2, 4] = c[4, 2] = 0.30    # (r_2, chi_2) = rho_2
    w = np.linalg.eigvalsh(c)
    assert w.min() > 0.05
    return c.tolist()


def _c5_uniforms():
    """256 uniforms of RandomStream(7).split(99) (rng.cpp:69-72), restated."""
    import oracle_api  # test infrastructure: the restated RNG

    R = oracle_api.restatement()
    return [float(x) for x in R.uniforms(R.key(7, 99), 0, 256)]


def case(name):
    if name == "minimal":
        j = _load("minimal.json")
        j["simulation"] = {"paths": 64, "replicas": 2}
        return j
    if name == "c1":
        desk = _load("desk.json")
        j = copy.deepcopy(desk)
        j["model"]["economies"] = desk["model"]["economies"][:1]
        j["model"]["clients"] = desk["model"]["clients"][:2]
        j["grid"] = {"pricing_steps": 50, "substeps": 25, "dt_years": 1.0}
        j["book"] = {"generate": {"count": 10, "notional_min": 1.0, "notional_max": 25.0}}
        j["simulation"] = {"paths": 1024, "replicas": 16}
        j["training"]["width"] = 32
        return j
    if name == "desk_corr":
        j = _load("desk.json")
        j["model"]["brownian_correlation"] = _desk_corr()
        j["grid"] = {"pricing_steps": 12, "substeps": 4, "dt_years": 0.5}
        j["simulation"] = {"paths": 40, "replicas": 8}
        return j
    if name == "c2":
        j = _load("paper_shape.json")
        j["grid"] = {"pricing_steps": 100, "substeps": 25, "dt_years": 0.25}
        j["simulation"] = {"paths": 16384, "replicas": 128}
        return j
    if name == "c5":
        # paper_shape economies, 64 clients with CIR parameters drawn
        # uniformly (alpha [0.3,0.7], delta [0.02,0.08], nu [0.05,0.15], gamma0
        # [0.01,0.06]) from RandomStream(7).split(99), 500 swaps, M=2^17, N=2^8.
        j = _load("paper_shape.json")
        u = _c5_uniforms()
        j["model"]["clients"] = [
            {"alpha": 0.3 + 0.4 * u[4 * c], "delta": 0.02 + 0.06 * u[4 * c + 1],
             "nu": 0.05 + 0.10 * u[4 * c + 2], "gamma0": 0.01 + 0.05 * u[4 * c + 3]} for c in range(64)]
        j["grid"] = {"pricing_steps": 100, "substeps": 25, "dt_years": 0.25}
        j["simulation"] = {"paths": 131072, "replicas": 256}
        return j
    if name == "c2_annual":
        j = case("c2")
        j["grid"]["dt_years"] = 1.0
        return j
    raise KeyError(name)


def text(name, **sim):
    j = case(name)
    if sim:
        j["simulation"] = dict(j["simulation"], **sim)
    return json.dumps(j)


def oracle_model(cfg):
    """PipelineConfig -> the dict taken by tests/oracle_api.py."""
    return dict(rates=cfg.rates, fx=cfg.fx, credit=cfg.credit,
                corr=None if cfg.correlation is None else cfg.correlation,
                n_steps=cfg.n_steps, substeps=cfg.substeps, dt=cfg.dt)


def twin_block(O, cfg, m, book, mk, st, step):
    """twin_labels at `step` (key seed/2/4/step) and the twin estimators on a
    fixed synthetic prediction; NaN where the reference raises numeric_error."""
    t1, t2 = O.twin_labels(m, book, step, mk, st, O.key(cfg.seed, 2, 4, step))
    pred = twin_prediction(t1, t2)
    N = st.shape[1]
    stats = []
    for block in (1, N):
        stats += list(O.twin_l2_error(pred, t1, t2, block))
    try:
        stats.append(O.twin_relative_rmse(pred, t1, t2))
    except Exception:  # OracleError: numeric_error (degenerate E[xi1 xi2])
        stats.append(float("nan"))
    stats += [O.twin_relative_rmse_std_error(pred, t1, t2, b) for b in (1, N)]
    return t1, t2, np.array(stats)


def twin_prediction(t1, t2):
    wiggle = 1.0 + 0.1 * np.sin(np.arange(t1.size).reshape(t1.shape))
    return np.mean(t1) * wiggle  # a path-blind prediction: the twin L2 is then positive
