"""On-disk formats: book CSV (portfolio.cpp:176-226)
against the compiled reference's writer, and the HCVAMDL1 model file
(regressor.cpp:397-481) / HCVAMKT1 market dump (pipeline.cpp:371-442) against
independent writers restated from the reference's byte layout."""
import ctypes as C
import os
import struct
import tempfile

import numpy as np
import pytest

import cases
import oracle_api
import paper_2211_17005_b200 as hcva
from paper_2211_17005_b200 import regression as rg


def test_book_csv_round_trip_and_reference_bytes():
    cfg = hcva.parse_config(cases.text("c2"))
    m = cases.oracle_model(cfg)
    R = oracle_api.restatement()
    root = R.key(cfg.seed)
    book = R.generate_book(m, 40, 1.0, 100.0, R.split(root, 0))
    with tempfile.TemporaryDirectory() as d:
        ours = os.path.join(d, "ours.csv")
        hcva.save_book_csv(ours, book)
        back = hcva.load_book_csv(ours, cfg)
        assert back.tobytes() == np.ascontiguousarray(book, dtype=hcva.SWAP_DTYPE).tobytes()
        F = oracle_api.reference()
        if F is None:
            pytest.skip("compiled reference not built here")
        theirs = os.path.join(d, "ref.csv")
        b = np.ascontiguousarray(book, dtype=hcva.SWAP_DTYPE)
        F._check(F.lib.or_save_book_csv(theirs.encode(), b.ctypes.data_as(C.c_void_p), len(b)))
        assert open(ours, "rb").read() == open(theirs, "rb").read()


def model_file_bytes(seed, config_hash, steps, h, u, d, act):
    """TrainedModelSequence::save (regressor.cpp:435-452) restated: Eigen writes
    matrices as (int64 rows, int64 cols, column-major doubles)."""
    out = [b"HCVAMDL1", struct.pack("<I", 1), struct.pack("<Q", seed), struct.pack("<i", len(steps)),
           struct.pack("<I", len(config_hash)), config_hash.encode()]

    def mat(a):
        a = np.atleast_2d(np.asarray(a, dtype=np.float64))
        return struct.pack("<qq", *a.shape) + a.tobytes(order="F")

    fin = [d] + [u] * h
    fout = [u] * h + [1]
    for p, mean, scale in steps:
        out += [struct.pack("<i", h + 1), struct.pack("<i", act), struct.pack("<d", p[-1])]
        off, Ws, Bs = 0, [], []
        for l in range(h + 1):
            Ws.append(p[off:off + fout[l] * fin[l]].reshape(fout[l], fin[l]))
            off += fout[l] * fin[l]
            Bs.append(p[off:off + fout[l]].reshape(-1, 1))
            off += fout[l]
        out += [mat(w) for w in Ws] + [mat(b) for b in Bs] + [mat(mean.reshape(-1, 1)), mat(scale.reshape(-1, 1))]
    return b"".join(out)


def market_dump_bytes(sim, seed, dt, substeps):
    """save_market (pipeline.cpp:382-406) restated over the exported AoS block."""
    mk = sim.market_arrays()
    M, n1, E = mk["rates"].shape
    Cn = mk["intens"].shape[2]
    head = b"HCVAMKT1" + struct.pack("<IQiiiiidi", 1, seed, M, n1 - 1, E, Cn, 0, dt, substeps)
    rows = np.concatenate([mk["rates"], mk["fx"], mk["intens"], mk["lagged"], mk["disc"][:, :, None],
                           mk["hazard"]], axis=2)
    return head + np.ascontiguousarray(rows, dtype="<f8").tobytes()


@pytest.mark.gpu
def test_model_file_bytes_and_round_trip():
    cfg = hcva.parse_config(cases.text("desk_corr"))
    t = cfg.training
    t.width, t.n_batches, t.epochs = 16, 8, 4
    book = hcva.generate_book(cfg)
    sim = hcva.simulate_set(cfg, book, 40, 8, hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM))
    models = rg.backward_learn(sim, t)
    steps = [models.get(i)[:3] for i in range(1, models.n_steps + 1)]
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "models.bin")
        models.save(path, seed=cfg.seed, config_hash="abc123")
        want = model_file_bytes(cfg.seed, "abc123", steps, t.hidden_layers, t.width, models.input_dim, 0)
        assert open(path, "rb").read() == want
        back = rg.load_models(path)
        assert back.seed == cfg.seed and back.config_hash == "abc123" and back.n_steps == models.n_steps
        for i in range(1, models.n_steps + 1):
            for a, b in zip(back.get(i)[:3], models.get(i)[:3]):
                assert np.array_equal(a, b)
            assert np.array_equal(back.predict(i, sim), models.predict(i, sim))
        # A file from the restated writer with other values loads as written.
        rng = np.random.default_rng(1)
        alt = [(rng.standard_normal(p.size), rng.random(m.size), 1 + rng.random(s.size)) for p, m, s in steps]
        with open(path, "wb") as f:
            f.write(model_file_bytes(7, "", alt, t.hidden_layers, t.width, models.input_dim, 0))
        back = rg.load_models(path)
        for i, (p, m, s) in enumerate(alt, start=1):
            got = back.get(i)
            assert np.array_equal(got[0], p) and np.array_equal(got[1], m) and np.array_equal(got[2], s)
        with open(path, "wb") as f:
            f.write(want[:-9])
        with pytest.raises(hcva.NumericError):
            rg.load_models(path)
        with open(path, "wb") as f:
            f.write(b"HCVAMDL2" + want[8:])
        with pytest.raises(hcva.ConfigError):
            rg.load_models(path)


@pytest.mark.gpu
def test_market_dump_bytes_and_reload():
    cfg = hcva.parse_config(cases.text("desk_corr"))
    book = hcva.generate_book(cfg)
    stream = hcva.RandomStream(cfg.seed).split(hcva.K_TRAIN_SIM)
    sim = hcva.simulate_set(cfg, book, 40, 8, stream)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "market.bin")
        sim.save_market(path, seed=cfg.seed)
        assert open(path, "rb").read() == market_dump_bytes(sim, cfg.seed, cfg.dt, cfg.substeps)
        back = hcva.load_market(cfg, path)
        assert back.seed == cfg.seed
        for k, v in sim.market_arrays().items():
            assert np.array_equal(back.market_arrays()[k], v), k
        # The loaded block runs the rest of the path: same defaults and cube.
        hcva.sample_default_block(back, 8, stream.split(1))
        hcva.build_mtm_cube(back, book)
        assert np.array_equal(back.default_steps(), sim.default_steps())
        assert np.array_equal(back.cube_values(), sim.cube_values())
        bad = hcva.parse_config(cases.text("c1"))
        with pytest.raises(hcva.ContractError):
            hcva.load_market(bad, path)
