"""C-ABI boundary checks that need no GPU: the library builds for sm_100a,
loads, exports every symbol include/hcva_gpu.h declares, and its host-side
entry points (book generation, par rates, Cholesky, error mapping) agree with
the oracle bit for bit."""
import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import cases
import oracle_api
import paper_2211_17005_b200 as hcva
from paper_2211_17005_b200 import _lib

HEADER = os.path.join(oracle_api.ROOT, "include", "hcva_gpu.h")


def declared_symbols():
    text = open(HEADER).read()
    return sorted(set(re.findall(r"\b(hcva_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    path = _lib.build()
    L = C.CDLL(path)
    syms = declared_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.EXPORTED) == syms


def test_library_is_sm100a_only():
    out = subprocess.run(["cuobjdump", "--list-elf", _lib.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert not re.search(r"sm_(?!100a)\d+", out)


def test_generate_book_bit_exact_vs_golden():
    for name in ("c1", "c2", "desk_corr"):
        z = np.load(f"{oracle_api.ROOT}/tests/golden/{name}.npz")
        cfg = hcva.parse_config(str(z["config"]))
        book = hcva.generate_book(cfg)
        ref = z["book"]
        for f in ref.dtype.names:
            assert np.array_equal(book[f], ref[f]), (name, f)


def test_par_zc_cholesky_match_oracle():
    R = oracle_api.restatement()
    cfg = hcva.parse_config(cases.text("desk_corr"))
    for v in cfg.rates:
        for mat in (1.0, 3.5, 12.0):
            assert hcva.par_rate(mat, 0.5, v) == R.par_rate(mat, 0.5, v)
        for tau in (0.0, 0.25, 7.0):
            assert hcva.zc_price(0.031, tau, v) == R.zc_price(0.031, tau, v)
    chol = hcva.cholesky(cfg)
    L = np.linalg.cholesky(np.array(cfg.correlation))
    assert np.allclose(chol, L, atol=1e-13)


def test_errors_map_to_reference_exception_types():
    cfg = hcva.parse_config(cases.text("desk_corr"))
    d = cfg.n_factors
    corr = np.eye(d)
    corr[1, 3] = corr[3, 1] = -0.25
    corr[2, 4] = corr[4, 2] = 0.30
    corr[0, 5] = corr[5, 0] = 0.95
    corr[0, 6] = corr[6, 0] = 0.95
    corr[5, 6] = corr[6, 5] = -0.9
    cfg.correlation = corr
    with pytest.raises(hcva.ConfigError, match="leading minor"):
        hcva.cholesky(cfg)
    with pytest.raises(hcva.ContractError):
        hcva.par_rate(3.3, 1.0, cfg.rates[0])
    with pytest.raises(hcva.ConfigError):
        hcva.parse_config("{ broken")
    bad = hcva.parse_config(cases.text("minimal"))
    bad.training.n_batches = 7
    with pytest.raises(hcva.ConfigError):
        bad.validate()
