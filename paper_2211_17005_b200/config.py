"""Pipeline configuration: the reference's JSON schema (proj/src/config.cpp:46-197).

Host-side only; it produces the model / grid / book descriptions handed to
the C ABI.  Defaults are the reference's (config.cpp:101-172).
"""
from __future__ import annotations

import ctypes as C
import json
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib


@dataclass
class TrainConfig:  # regressor.hpp:33-44
    epochs: int = 8
    n_batches: int = 32
    learning_rate: float = 0.001
    adam: bool = True
    hidden_layers: int = 2
    width: int = 64
    activation: str = "tanh"
    seed: int = 0
    ridge: float = 1e-8


@dataclass
class PipelineConfig:  # config.hpp:61-76
    rates: np.ndarray            # (E, 4) a, b, sigma, r0
    fx: np.ndarray               # (E-1, 3) sigma, rho, chi0
    credit: np.ndarray           # (Cc+1, 4) alpha, delta, nu, gamma0 (bank first)
    correlation: Optional[np.ndarray] = None
    n_steps: int = 1
    substeps: int = 1
    dt: float = 1.0
    book_file: Optional[str] = None
    book_count: int = 10
    notional_min: float = 1.0
    notional_max: float = 100.0
    paths: int = 256
    replicas: int = 1
    training: TrainConfig = field(default_factory=TrainConfig)
    label_kind: str = "defaults"
    collect_qr_trace: bool = False
    twin: bool = True
    nested: bool = False
    inner_paths: int = 0
    validation_paths: int = 512
    nested_states: int = 128
    validation_steps_list: List[int] = field(default_factory=list)
    seed: int = 0
    output_dir: str = "out"

    # -- derived ---------------------------------------------------------
    @property
    def n_economies(self) -> int:
        return self.rates.shape[0]

    @property
    def n_clients(self) -> int:
        return self.credit.shape[0] - 1

    @property
    def n_factors(self) -> int:
        return 2 * self.n_economies - 1 + self.n_clients + 1

    def set_scale(self, m: int, n: int) -> None:
        self.paths, self.replicas = m, n

    def validate(self) -> None:  # config.cpp:181-197
        if self.paths < 1 or self.replicas < 1:
            raise _lib.ConfigError("config: simulation paths and replicas must be >= 1")
        if (self.paths * self.replicas) % self.training.n_batches != 0:
            raise _lib.ConfigError("config: batch count must divide M*N")
        if self.label_kind not in ("defaults", "intensity"):
            raise _lib.ConfigError("config: label_kind must be 'defaults' or 'intensity'")
        for s in self.validation_steps_list:
            if s < 1 or s > self.n_steps:
                raise _lib.ConfigError("config: validation steps must lie in {1..n}")

    def validation_steps(self) -> List[int]:  # config.cpp:199-205
        if self.validation_steps_list:
            return list(self.validation_steps_list)
        n = self.n_steps
        out = []
        for s in (max(1, n // 4), max(1, n // 2), max(1, (3 * n) // 4)):
            if not out or out[-1] != s:
                out.append(s)
        return out

    def to_model(self):
        """ctypes hcva_model + hcva_grid; keeps the backing arrays alive on the result."""
        E, Cn = self.n_economies, self.credit.shape[0]
        rates = (_lib.Vasicek * E)(*[_lib.Vasicek(*map(float, r)) for r in self.rates])
        fx = (_lib.Fx * max(E - 1, 1))(*[_lib.Fx(*map(float, f)) for f in self.fx])
        credit = (_lib.Cir * Cn)(*[_lib.Cir(*map(float, c)) for c in self.credit])
        corr = None
        if self.correlation is not None:
            corr = np.ascontiguousarray(self.correlation, dtype=np.float64)
        m = _lib.Model(E, Cn - 1, rates, fx, credit,
                       corr.ctypes.data_as(_lib.dptr) if corr is not None else _lib.dptr())
        m._keep = (rates, fx, credit, corr)
        g = _lib.Grid(self.n_steps, self.substeps, self.dt)
        return m, g


def parse_config(text: str) -> PipelineConfig:  # config.cpp:46-172
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise _lib.ConfigError(f"config: invalid JSON: {e}") from None
    try:
        jm = j["model"]
        rates, fx = [], []
        for idx, je in enumerate(jm["economies"]):
            rates.append([je["a"], je["b"], je["sigma"], je["r0"]])
            if idx > 0:
                f = je["fx"]
                fx.append([f["sigma"], f["rho"], f["chi0"]])
        credit = [[jm["bank"][k] for k in ("alpha", "delta", "nu", "gamma0")]]
        for jc in jm["clients"]:
            credit.append([jc[k] for k in ("alpha", "delta", "nu", "gamma0")])
        corr = jm.get("brownian_correlation")
        jg = j["grid"]
        cfg = PipelineConfig(
            rates=np.array(rates, dtype=np.float64),
            fx=np.array(fx, dtype=np.float64).reshape(-1, 3),
            credit=np.array(credit, dtype=np.float64),
            correlation=None if corr is None else np.array(corr, dtype=np.float64),
            n_steps=int(jg["pricing_steps"]),
            substeps=int(jg.get("substeps", 1)),
            dt=float(jg.get("dt_years", 1.0)),
            seed=int(j.get("seed", 0)),
            output_dir=j.get("output_dir", "out"),
        )
    except (KeyError, TypeError) as e:
        raise _lib.ConfigError(f"config: missing or malformed key {e}") from None
    jb = j.get("book", {})
    if "file" in jb:
        cfg.book_file = jb["file"]
    elif "generate" in jb:
        gg = jb["generate"]
        cfg.book_count = int(gg.get("count", 10))
        cfg.notional_min = float(gg.get("notional_min", 1.0))
        cfg.notional_max = float(gg.get("notional_max", 100.0))
    if "simulation" in j:
        cfg.paths = int(j["simulation"].get("paths", 256))
        cfg.replicas = int(j["simulation"].get("replicas", 1))
    if "training" in j:
        jt = j["training"]
        t = cfg.training
        t.epochs = int(jt.get("epochs", 8))
        t.n_batches = int(jt.get("batches", 32))
        t.learning_rate = float(jt.get("learning_rate", 0.001))
        t.adam = jt.get("optimizer", "adam") == "adam"
        t.hidden_layers = int(jt.get("hidden_layers", 2))
        t.width = int(jt.get("width", 64))
        t.activation = jt.get("activation", "tanh")
        if t.activation not in ("tanh", "sigmoid", "softplus", "relu"):
            raise _lib.ConfigError(f"unknown activation: {t.activation}")
        t.ridge = float(jt.get("ridge", 1e-8))
        cfg.label_kind = jt.get("label_kind", "defaults")
        cfg.collect_qr_trace = bool(jt.get("collect_qr_trace", False))
    cfg.training.seed = cfg.seed
    if "validation" in j:
        jv = j["validation"]
        cfg.twin = bool(jv.get("twin", True))
        cfg.nested = bool(jv.get("nested", False))
        cfg.inner_paths = int(jv.get("inner_paths", 0))
        cfg.validation_paths = int(jv.get("paths", 512))
        cfg.nested_states = int(jv.get("nested_states", 128))
        cfg.validation_steps_list = [int(s) for s in jv.get("steps", [])]
    return cfg


def load_config(path: str) -> PipelineConfig:
    try:
        with open(path) as f:
            return parse_config(f.read())
    except OSError:
        raise _lib.ConfigError(f"config: cannot open {path}") from None
