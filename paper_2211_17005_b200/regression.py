"""Backward MLP regression (regressor.hpp:33-139) on the GPU, over the C ABI.

    models = backward_learn(sim, cfg)            # Alg. 2 over every pricing step
    params, mean, scale, report = models.get(5)  # StepModel of step 5
    pred = models.predict(5, validation_sim)     # TrainedModelSequence::predict
"""
from __future__ import annotations

import ctypes as C
from typing import Dict, Optional, Tuple

import numpy as np

from . import _lib
from .config import PipelineConfig, TrainConfig
from .engine import Context, SimulationSet, context

ACTIVATIONS = {"tanh": 0, "sigmoid": 1, "softplus": 2, "relu": 3}


def train_cfg(t: TrainConfig) -> _lib.TrainCfg:
    if t.activation not in ACTIVATIONS:
        raise _lib.ConfigError(f"unknown activation: {t.activation}")
    return _lib.TrainCfg(t.epochs, t.n_batches, t.hidden_layers, t.width, ACTIVATIONS[t.activation],
                         int(bool(t.adam)), t.learning_rate, t.ridge, t.seed)


def net_size(t: TrainConfig, input_dim: int) -> int:
    n = C.c_int()
    _lib.check(_lib.lib().hcva_net_size(C.byref(train_cfg(t)), input_dim, C.byref(n)))
    return n.value


def init_network(t: TrainConfig, input_dim: int, key: int) -> np.ndarray:
    """init_network (regressor.cpp:172-189) from a stream key (mu = 0)."""
    p = np.zeros(net_size(t, input_dim))
    _lib.check(_lib.lib().hcva_init_network(C.byref(train_cfg(t)), input_dim, key, p.ctypes.data_as(_lib.dptr)))
    return p


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def quadratic_loss(t: TrainConfig, params: np.ndarray, x: np.ndarray, y: np.ndarray, head: bool = False,
                   ctx: Optional[Context] = None) -> Tuple[float, np.ndarray]:
    """quadratic_loss (regressor.cpp:115-158): (loss, gradients in the flat layout)."""
    ctx = ctx or context()
    x, y, params = _f64(x), _f64(y), _f64(params)
    g = np.zeros_like(params)
    loss = C.c_double()
    _lib.check(_lib.lib().hcva_quadratic_loss(ctx.handle, C.byref(train_cfg(t)), x.shape[1],
                                              params.ctypes.data_as(_lib.dptr), int(head),
                                              x.ctypes.data_as(_lib.dptr), y.ctypes.data_as(_lib.dptr),
                                              x.shape[0], C.byref(loss), g.ctypes.data_as(_lib.dptr)))
    return loss.value, g


def sim_quadratic_loss(sim: SimulationSet, t: TrainConfig, step: int, params: np.ndarray, mean: np.ndarray,
                       scale: np.ndarray, head: bool = False, rows: Optional[Tuple[int, int]] = None,
                       label_kind: str = "defaults") -> Tuple[float, np.ndarray]:
    """quadratic_loss (regressor.cpp:115-158) on the label source's rows of a simulated set at `step`
    (features standardised with mean / scale) through the kernels backward_learn runs on it."""
    params, mean, scale = _f64(params), _f64(mean), _f64(scale)
    b0, b1 = rows if rows is not None else (0, sim.n_paths * sim.n_replicas)
    g = np.zeros_like(params)
    loss = C.c_double()
    kind = {"defaults": 0, "intensity": 1}[label_kind]
    _lib.check(_lib.lib().hcva_sim_quadratic_loss(sim.handle, C.byref(train_cfg(t)), int(step), kind,
                                                  params.ctypes.data_as(_lib.dptr), mean.ctypes.data_as(_lib.dptr),
                                                  scale.ctypes.data_as(_lib.dptr), int(head), int(b0), int(b1),
                                                  C.byref(loss), g.ctypes.data_as(_lib.dptr)))
    return loss.value, g


def sgd_timing(sim: SimulationSet, t: TrainConfig, step: int, steps: int = 50, label_kind: str = "defaults"):
    """Mean ms of [SGD step, gradient kernels, optimizer] and whether the split kernels ran (hcva_diag_sgd_timing)."""
    out = np.zeros(5)
    kind = {"defaults": 0, "intensity": 1}[label_kind]
    _lib.check(_lib.lib().hcva_diag_sgd_timing(sim.handle, C.byref(train_cfg(t)), int(step), kind, int(steps),
                                               out.ctypes.data_as(_lib.dptr)))
    return dict(step_ms=out[0], gradient_ms=out[1], optimizer_ms=out[2], split=bool(out[3]),
                fused_step_ms=out[4] if out[4] > 0 else None)


def forward(t: TrainConfig, params: np.ndarray, x: np.ndarray, ctx: Optional[Context] = None) -> np.ndarray:
    """forward (regressor.cpp:97-113) with the positive head on, on standardised rows: predictions."""
    ctx = ctx or context()
    x, params = _f64(x), _f64(params)
    out = np.zeros(x.shape[0])
    _lib.check(_lib.lib().hcva_forward(ctx.handle, C.byref(train_cfg(t)), x.shape[1], params.ctypes.data_as(_lib.dptr),
                                       x.ctypes.data_as(_lib.dptr), x.shape[0], out.ctypes.data_as(_lib.dptr)))
    return out


def refit_output_layer(t: TrainConfig, params: np.ndarray, x: np.ndarray, y: np.ndarray,
                       ctx: Optional[Context] = None) -> np.ndarray:
    """refit_output_layer (regressor.cpp:191-213): a copy of params with the output layer refit."""
    ctx = ctx or context()
    x, y = _f64(x), _f64(y)
    p = np.array(params, dtype=np.float64)
    _lib.check(_lib.lib().hcva_refit_output_layer(ctx.handle, C.byref(train_cfg(t)), x.shape[1],
                                                  p.ctypes.data_as(_lib.dptr), x.ctypes.data_as(_lib.dptr),
                                                  y.ctypes.data_as(_lib.dptr), x.shape[0]))
    return p


def train_base(t: TrainConfig, x: np.ndarray, y: np.ndarray, init: np.ndarray, ctx: Optional[Context] = None):
    """train_base (regressor.cpp:265-347) with contiguous batches: (best params, report)."""
    ctx = ctx or context()
    x, y, init = _f64(x), _f64(y), _f64(init)
    best = np.zeros_like(init)
    losses = np.zeros(t.epochs)
    bl, be = C.c_double(), C.c_int()
    _lib.check(_lib.lib().hcva_train_base(ctx.handle, C.byref(train_cfg(t)), x.shape[1], x.ctypes.data_as(_lib.dptr),
                                          y.ctypes.data_as(_lib.dptr), x.shape[0], init.ctypes.data_as(_lib.dptr),
                                          best.ctypes.data_as(_lib.dptr), losses.ctypes.data_as(_lib.dptr),
                                          C.byref(bl), C.byref(be)))
    return best, dict(epoch_losses=losses, best_loss=bl.value, best_epoch=be.value)


class Models:
    """TrainedModelSequence (regressor.hpp:120-131), device resident."""

    def __init__(self, handle, ctx: Context):
        self.handle, self.ctx = handle, ctx
        info = (C.c_int * 4)()
        _lib.check(_lib.lib().hcva_models_info(handle, info))
        self.n_steps, self.input_dim, self.n_params, self.epochs = list(info)

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().hcva_models_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    def get(self, step: int):
        p, mean, scale = np.zeros(self.n_params), np.zeros(self.input_dim), np.zeros(self.input_dim)
        losses = np.zeros(self.epochs)
        bl, be = C.c_double(), C.c_int()
        d = lambda a: a.ctypes.data_as(_lib.dptr)  # noqa: E731
        _lib.check(_lib.lib().hcva_models_get(self.handle, step, d(p), d(mean), d(scale), d(losses), C.byref(bl),
                                              C.byref(be)))
        return p, mean, scale, dict(epoch_losses=losses, best_loss=bl.value, best_epoch=be.value)

    def predict(self, step: int, sim: SimulationSet) -> np.ndarray:
        out = np.zeros(sim.n_paths * sim.n_replicas)
        _lib.check(_lib.lib().hcva_predict(self.handle, sim.handle, step, out.ctypes.data_as(_lib.dptr)))
        return out

    def save(self, path: str, seed: int = 0, config_hash: str = "") -> None:
        """TrainedModelSequence::save (regressor.cpp:435-452): the HCVAMDL1 file."""
        _lib.check(_lib.lib().hcva_models_save(self.handle, path.encode(), seed, config_hash.encode()))


def load_models(path: str, ctx: Optional[Context] = None) -> Models:
    """TrainedModelSequence::load (regressor.cpp:454-481); ``.seed`` / ``.config_hash`` set."""
    ctx = ctx or context()
    h = C.c_void_p()
    seed = C.c_uint64()
    buf = C.create_string_buffer(4096)
    _lib.check(_lib.lib().hcva_models_load(ctx.handle, path.encode(), C.byref(seed), buf, len(buf), C.byref(h)))
    m = Models(h, ctx)
    m.seed, m.config_hash = seed.value, buf.value.decode()
    return m


def backward_learn(sim: SimulationSet, t: TrainConfig, label_kind: str = "defaults", comm=None,
                   qr_probe=None) -> Models:
    """backward_learn (regressor.cpp:354-395) over the label source of make_label_source.

    With ``comm`` (a ``dist.Comm`` of world G) ``sim`` is this rank's interleaved
    shard (``dist.shard_spec``) and every cross-rank sum is a rank-ordered
    allgather of FP64 partials: all ranks end with the same networks.

    With ``qr_probe`` (the reference's probe stream, root.split(kTrainSim).split(2))
    the Q/R trace of collect_qr_trace is recorded: ``models.qr_trace`` is an
    array of rows (step, epoch, Q, R) in training order."""
    kind = {"defaults": 0, "intensity": 1}.get(label_kind)
    if kind is None:
        raise _lib.ConfigError("config: label_kind must be 'defaults' or 'intensity'")
    h = C.c_void_p()
    if qr_probe is not None:
        if comm is not None:
            raise _lib.ContractError("Q/R probe: single-GPU runs only")
        trace = np.zeros((sim.n_steps * t.epochs, 4))
        _lib.check(_lib.lib().hcva_backward_learn_qr(sim.handle, C.byref(train_cfg(t)), kind, qr_probe.key,
                                                     trace.ctypes.data_as(_lib.dptr), C.byref(h)))
        models = Models(h, sim.ctx)
        models.qr_trace = trace
        return models
    _lib.check(_lib.lib().hcva_backward_learn_dist(sim.handle, C.byref(train_cfg(t)), kind,
                                                   comm.handle if comm is not None else None, C.byref(h)))
    return Models(h, sim.ctx)


def probe_block(sim: SimulationSet, stream, label_kind: str = "defaults"):
    """The Q/R probe's two extra replicas per path (pipeline.cpp:79-81) and their labels:
    (steps (M, 2, Cn) uint16, labels (n+1, M, 2))."""
    kind = {"defaults": 0, "intensity": 1}[label_kind]
    st = np.zeros((sim.n_paths, 2, sim.n_credit), dtype=np.uint16)
    lab = np.zeros((sim.n_steps + 1, sim.n_paths, 2))
    _lib.check(_lib.lib().hcva_probe_block(sim.handle, stream.key, kind, st.ctypes.data_as(C.POINTER(C.c_uint16)),
                                           lab.ctypes.data_as(_lib.dptr)))
    return st, lab


def estimate_qr(g1, g2) -> Dict[str, float]:
    """estimate_qr (planner.cpp:11-70)."""
    a = np.ascontiguousarray(g1, dtype=np.float64)
    b = np.ascontiguousarray(g2, dtype=np.float64)
    if a.size != b.size:
        raise _lib.ContractError("estimate_qr: pair length mismatch")
    out = np.zeros(6)
    _lib.check(_lib.lib().hcva_estimate_qr(context().handle, a.ctypes.data_as(_lib.dptr), b.ctypes.data_as(_lib.dptr), a.size,
                                           out.ctypes.data_as(_lib.dptr)))
    return dict(q=out[0], r=out[1], total=out[2], n_pairs=int(out[3]), q_std_error=out[4], r_std_error=out[5])


def percentile_table(models: Models, validation: SimulationSet) -> Dict[int, Dict[str, float]]:
    """percentile_table (pipeline.cpp:138-156): out-of-sample mean and percentile bands per step,
    predicted, sorted and reduced on the GPU."""
    out = np.zeros((models.n_steps, 6))
    _lib.check(_lib.lib().hcva_percentile_table(models.handle, validation.handle, out.ctypes.data_as(_lib.dptr)))
    return {int(r[0]): dict(mean=r[1], p1=r[2], p2_5=r[3], p97_5=r[4], p99=r[5]) for r in out}
