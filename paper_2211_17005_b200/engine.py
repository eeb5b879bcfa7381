"""Python surface of the engine, mirroring the reference's pybind module
(proj/python/hiercva_module.cpp:45-180) on top of the C ABI.

    import paper_2211_17005_b200 as hcva
    cfg = hcva.load_config("paper_shape.json")
    market, defaults, cube = hcva.simulate(cfg, paths, replicas)   # on the GPU
    xi = hcva.defaults_label(step, cfg, market, defaults)          # (M, N)
    f  = hcva.features(step, market, defaults)                     # (M*N, p+q)

Everything below dispatches to libhcva_gpu.so; nothing here computes on the
CPU beyond host-side bookkeeping.
"""
from __future__ import annotations

import ctypes as C
import threading
from typing import Dict, Optional, Tuple

import numpy as np

from . import _lib
from .config import PipelineConfig

# Stream lineage keys of the pipeline phases (pipeline.hpp:26-31).
K_BOOK, K_TRAIN_SIM, K_VALIDATION_SIM, K_ARD = 0, 1, 2, 3

SWAP_DTYPE = np.dtype([("economy", "<i4"), ("client", "<i4"), ("notional", "<f8"),
                       ("tenor", "<f8"), ("maturity", "<f8"), ("fixed_rate", "<f8")], align=True)


class Context:
    """One GPU, one CUDA stream (hcva_ctx)."""

    def __init__(self, device: int = 0):
        L = _lib.lib()
        h = C.c_void_p()
        _lib.check(L.hcva_ctx_create(device, C.byref(h)))
        self.handle = h
        self.device = device

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _lib.check(_lib.lib().hcva_ctx_stream(self.handle, C.byref(s)))
        return s.value or 0

    def synchronize(self) -> None:
        _lib.check(_lib.lib().hcva_ctx_synchronize(self.handle))

    def launch_count(self) -> int:
        v = C.c_uint64()
        _lib.check(_lib.lib().hcva_ctx_launch_count(self.handle, C.byref(v)))
        return v.value

    def close(self) -> None:
        if self.handle:
            _lib.lib().hcva_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_ctx_lock = threading.Lock()
_contexts: Dict[int, Context] = {}


def context(device: int = 0) -> Context:
    with _ctx_lock:
        if device not in _contexts:
            _contexts[device] = Context(device)
        return _contexts[device]


class RandomStream:
    """Key-level mirror of hiercva::RandomStream (rng.hpp:16-52); draws run on the GPU."""

    def __init__(self, seed: int = 0, _key: Optional[int] = None):
        L = _lib.lib()
        self.key = int(_key) if _key is not None else int(L.hcva_rng_root_key(seed))
        self.pos = 0

    def split(self, k: int) -> "RandomStream":
        return RandomStream(_key=_lib.lib().hcva_rng_split_key(self.key, int(k)))

    def _draw(self, n: int, kind: int, dtype) -> np.ndarray:
        out = np.zeros(n, dtype=dtype)
        if n:
            _lib.check(_lib.lib().hcva_rng_draw(context().handle, self.key, self.pos, n, kind,
                                                out.ctypes.data_as(C.c_void_p)))
        self.pos += n
        return out

    def u64(self, n: int) -> np.ndarray:
        return self._draw(n, 0, np.uint64)

    def uniforms(self, n: int) -> np.ndarray:
        return self._draw(n, 1, np.float64)

    def normals(self, n: int) -> np.ndarray:
        return self._draw(n, 2, np.float64)

    def exponentials(self, n: int) -> np.ndarray:
        return self._draw(n, 3, np.float64)


def _swaps(book: np.ndarray):
    book = np.ascontiguousarray(book, dtype=SWAP_DTYPE)
    return book, book.ctypes.data_as(C.POINTER(_lib.Swap))


def generate_book(cfg: PipelineConfig, stream: Optional[RandomStream] = None) -> np.ndarray:
    """generate_book (portfolio.cpp:149-174) from root.split(kBook) by default."""
    m, g = cfg.to_model()
    key = stream.key if stream is not None else RandomStream(cfg.seed).split(K_BOOK).key
    out = np.zeros(cfg.book_count, dtype=SWAP_DTYPE)
    _lib.check(_lib.lib().hcva_generate_book(C.byref(m), C.byref(g), cfg.book_count,
                                             cfg.notional_min, cfg.notional_max, key,
                                             out.ctypes.data_as(C.POINTER(_lib.Swap))))
    return out


def load_book_csv(path: str, cfg: PipelineConfig) -> np.ndarray:
    """load_book_csv (portfolio.cpp:176-212): economy,client,notional,tenor,maturity,rate|par."""
    rows = []
    with open(path) as f:
        first = True
        for line in f:
            line = line.strip()
            if not line:
                continue
            if first and line.startswith("economy"):
                first = False
                continue
            first = False
            parts = line.split(",")
            if len(parts) < 6:
                raise _lib.ConfigError(f"book: malformed row: {line}")
            e, c = int(parts[0]), int(parts[1])
            notional, tenor, maturity = float(parts[2]), float(parts[3]), float(parts[4])
            if parts[5] == "par":
                rate = par_rate(maturity, tenor, cfg.rates[e])
            else:
                rate = float(parts[5])
            rows.append((e, c, notional, tenor, maturity, rate))
    if not rows:
        raise _lib.ConfigError(f"book: no swaps in {path}")
    return np.array(rows, dtype=SWAP_DTYPE)


def save_book_csv(path: str, book: np.ndarray) -> None:
    """save_book_csv (portfolio.cpp:216-226): header + %d,%d,%.17g x4 rows."""
    with open(path, "w") as f:
        f.write("economy,client,notional,tenor,maturity,rate\n")
        for sw in np.asarray(book, dtype=SWAP_DTYPE):
            f.write("%d,%d,%.17g,%.17g,%.17g,%.17g\n" % (sw["economy"], sw["client"], sw["notional"], sw["tenor"],
                                                        sw["maturity"], sw["fixed_rate"]))


def load_market(cfg: PipelineConfig, path: str, ctx: Optional[Context] = None) -> "SimulationSet":
    """load_market (pipeline.cpp:408-442) into a set on the GPU (HCVAMKT1); ``.seed`` set."""
    ctx = ctx or context()
    m, g = cfg.to_model()
    h = C.c_void_p()
    seed = C.c_uint64()
    _lib.check(_lib.lib().hcva_market_load(ctx.handle, C.byref(m), C.byref(g), path.encode(), C.byref(seed),
                                           C.byref(h)))
    sim = SimulationSet(h, ctx)
    sim.seed = seed.value
    return sim


def resolve_book(cfg: PipelineConfig) -> np.ndarray:  # pipeline.cpp:57-61
    return load_book_csv(cfg.book_file, cfg) if cfg.book_file else generate_book(cfg)


def par_rate(maturity: float, tenor: float, vasicek) -> float:
    v = _lib.Vasicek(*map(float, vasicek))
    out = C.c_double()
    _lib.check(_lib.lib().hcva_par_rate(maturity, tenor, C.byref(v), C.byref(out)))
    return out.value


def zc_price(r: float, tau: float, vasicek) -> float:
    v = _lib.Vasicek(*map(float, vasicek))
    out = C.c_double()
    _lib.check(_lib.lib().hcva_zc_price(r, tau, C.byref(v), C.byref(out)))
    return out.value


def cholesky(cfg: PipelineConfig) -> np.ndarray:
    m, _ = cfg.to_model()
    d = cfg.n_factors
    out = np.zeros((d, d))
    _lib.check(_lib.lib().hcva_cholesky(C.byref(m), out.ctypes.data_as(_lib.dptr)))
    return out


class SimulationSet:
    """A simulated (market, defaults, cube) set resident on the GPU (hcva_sim).

    The three reference objects (MarketBlock, DefaultBlock, MtMCube) are views of
    this one handle: `market`, `defaults` and `cube` all return self so that
    `market, defaults, cube = simulate(...)` reads like the reference API.
    """

    def __init__(self, handle, ctx: Context):
        self.handle = handle
        self.ctx = ctx
        dims = (C.c_int * 8)()
        _lib.check(_lib.lib().hcva_sim_dims(handle, dims))
        (self.n_paths, self.n_steps, self.n_economies, self.n_credit, self.n_replicas,
         self.start_step, self.n_factors, self.substeps) = list(dims)
        self._market = None

    def __del__(self):
        try:
            if self.handle:
                _lib.lib().hcva_sim_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    @property
    def n_clients(self) -> int:
        return self.n_credit - 1

    # -- exports in the reference's AoS layouts --------------------------
    def market_arrays(self) -> Dict[str, np.ndarray]:
        if self._market is None:
            M, n1, E, Cn = self.n_paths, self.n_steps + 1, self.n_economies, self.n_credit
            out = dict(rates=np.zeros((M, n1, E)), fx=np.zeros((M, n1, E - 1)),
                       intens=np.zeros((M, n1, Cn)), lagged=np.zeros((M, n1, E)),
                       disc=np.zeros((M, n1)), hazard=np.zeros((M, n1, Cn)))
            p = lambda a: a.ctypes.data_as(C.c_void_p) if a.size else None  # noqa: E731
            _lib.check(_lib.lib().hcva_sim_export_market(
                self.handle, p(out["rates"]), p(out["fx"]), p(out["intens"]), p(out["lagged"]),
                p(out["disc"]), p(out["hazard"])))
            self._market = out
        return self._market

    def default_steps(self) -> np.ndarray:
        out = np.zeros((self.n_paths, self.n_replicas, self.n_credit), dtype=np.uint16)
        _lib.check(_lib.lib().hcva_sim_export_defaults(self.handle, out.ctypes.data_as(C.c_void_p)))
        return out

    def cube_values(self) -> np.ndarray:
        out = np.zeros((self.n_paths, self.n_steps + 1, self.n_clients))
        _lib.check(_lib.lib().hcva_sim_export_cube(self.handle, out.ctypes.data_as(C.c_void_p)))
        return out

    def save_market(self, path: str, seed: int = 0) -> None:
        """save_market (pipeline.cpp:371-406): the HCVAMKT1 dump of this set's market block."""
        _lib.check(_lib.lib().hcva_sim_save_market(self.handle, path.encode(), seed))

    def tie_counts(self) -> Tuple[int, int]:
        out = (C.c_uint64 * 2)()
        _lib.check(_lib.lib().hcva_sim_tie_counts(self.handle, out))
        return int(out[0]), int(out[1])

    # -- reference accessors (MarketBlock / DefaultBlock / MtMCube) --------
    def rate(self, k, i, e):
        return self.market_arrays()["rates"][k, i, e]

    def fx(self, k, i, e):
        return 1.0 if e == 0 else self.market_arrays()["fx"][k, i, e - 1]

    def intensity(self, k, i, c):
        return self.market_arrays()["intens"][k, i, c]

    def lagged_rate(self, k, i, e):
        return self.market_arrays()["lagged"][k, i, e]

    def discount(self, k, i):
        return self.market_arrays()["disc"][k, i]

    def hazard(self, k, i, c):
        return self.market_arrays()["hazard"][k, i, c]

    def default_step(self, k, l, c):
        return int(self.default_steps()[k, l, c])

    def indicator(self, k, l, i, c):
        return self.default_step(k, l, c) <= i

    def at(self, k, i, client):
        return self.cube_values()[k, i, client - 1]

    def state_at(self, k: int, i: int) -> Dict[str, np.ndarray]:
        """MarketState at (k, i) (market.cpp:100-113)."""
        mk = self.market_arrays()
        return dict(rates=mk["rates"][k, i].copy(), log_fx=np.log(mk["fx"][k, i]),
                    intens=mk["intens"][k, i].copy(), lagged=mk["lagged"][k, i].copy())

    def states_at(self, i: int, replica: int = 0) -> Tuple[Dict[str, np.ndarray], np.ndarray]:
        """MarketState of every path at step i and the clients' survival to i on
        `replica` -- the outer states of nested_cva (pipeline.cpp:276-288,
        validation.cpp:129-131): (states dict of (M, .) arrays, survived (M, Cc))."""
        mk = self.market_arrays()
        st = dict(rates=np.ascontiguousarray(mk["rates"][:, i]), log_fx=np.log(mk["fx"][:, i]),
                  intens=np.ascontiguousarray(mk["intens"][:, i]), lagged=np.ascontiguousarray(mk["lagged"][:, i]))
        surv = self.default_steps()[:, replica, 1:] > i
        return st, surv

    # -- labels and features -------------------------------------------
    def labels(self, step: int, kind: str = "defaults") -> np.ndarray:
        out = np.zeros((self.n_paths, self.n_replicas))
        _lib.check(_lib.lib().hcva_labels(self.handle, step, _kind(kind), out.ctypes.data_as(C.c_void_p)))
        return out

    def labels_all(self, kind: str = "defaults", to_host: bool = True) -> Optional[np.ndarray]:
        if not to_host:
            _lib.check(_lib.lib().hcva_labels_all(self.handle, _kind(kind), None))
            return None
        out = np.zeros((self.n_steps + 1, self.n_paths, self.n_replicas))
        _lib.check(_lib.lib().hcva_labels_all(self.handle, _kind(kind), out.ctypes.data_as(C.c_void_p)))
        return out

    def cva_profile(self, kind: str = "defaults") -> np.ndarray:
        """E[xi_i] for i = 0..n (mean label per step; out[0] = time-0 CVA)."""
        out = np.zeros(self.n_steps + 1)
        _lib.check(_lib.lib().hcva_cva_profile(self.handle, _kind(kind), out.ctypes.data_as(C.c_void_p)))
        return out

    def rerun(self, stream: "RandomStream", labels: Optional[str] = "defaults", event_slot: int = -1) -> None:
        """Asynchronous in-place re-simulation with new keys (stream.split(0/1))."""
        kind = -1 if labels is None else _kind(labels)
        _lib.check(_lib.lib().hcva_sim_rerun(self.handle, stream.split(0).key, stream.split(1).key, kind,
                                             event_slot))
        self._market = None

    def phase_times(self, event_slot: int) -> np.ndarray:
        ms = (C.c_float * 4)()
        _lib.check(_lib.lib().hcva_sim_phase_times(self.handle, event_slot, ms))
        return np.array(list(ms))

    def features(self, step: int) -> np.ndarray:
        E, Cn = self.n_economies, self.n_credit
        cols = (Cn - 1) + E + (E - 1) + (Cn - 1) + E
        out = np.zeros((self.n_paths * self.n_replicas, cols))
        _lib.check(_lib.lib().hcva_features(self.handle, step, out.ctypes.data_as(C.c_void_p)))
        return out


def _kind(kind: str) -> int:
    if kind == "defaults":
        return 0
    if kind == "intensity":
        return 1
    raise _lib.ConfigError("label_kind must be 'defaults' or 'intensity'")


def simulate_set(cfg: PipelineConfig, book: Optional[np.ndarray], n_paths: int, n_replicas: int,
                 stream: RandomStream, path_offset: int = 0, ctx: Optional[Context] = None,
                 shard: Optional[Tuple[int, int]] = None) -> SimulationSet:
    """simulate_set (pipeline.cpp:63-70): market from stream.split(0), defaults from stream.split(1).

    Local path k is global path ``path_offset + k``, or with ``shard = (blk, stride)``
    ``path_offset + (k // blk) * stride + k % blk`` (an interleaved multi-GPU shard,
    see ``dist.shard_spec``)."""
    ctx = ctx or context()
    m, g = cfg.to_model()
    h = C.c_void_p()
    if book is not None:
        bk, bp = _swaps(book)
        nsw = len(bk)
    else:
        bp, nsw = None, 0
    blk, stride = shard if shard else (0, 0)
    _lib.check(_lib.lib().hcva_simulate_set_sharded(ctx.handle, C.byref(m), C.byref(g), bp, nsw, n_paths,
                                                    path_offset, blk, stride, n_replicas, stream.split(0).key,
                                                    stream.split(1).key, C.byref(h)))
    return SimulationSet(h, ctx)


def simulate_market(cfg: PipelineConfig, n_paths: int, stream: RandomStream,
                    ctx: Optional[Context] = None) -> SimulationSet:
    """simulate_market (market.cpp:161-234): path k draws from stream.split(k)."""
    ctx = ctx or context()
    m, g = cfg.to_model()
    h = C.c_void_p()
    _lib.check(_lib.lib().hcva_simulate_set(ctx.handle, C.byref(m), C.byref(g), None, 0, n_paths, 0,
                                            0, stream.key, 0, C.byref(h)))
    return SimulationSet(h, ctx)


def simulate_conditional_market(cfg: PipelineConfig, state: Dict[str, np.ndarray], start_step: int,
                                horizon: int, n_inner: int, stream: RandomStream,
                                ctx: Optional[Context] = None) -> SimulationSet:
    """simulate_conditional_market (market.cpp:236-310): inner path l draws from stream.split(l)."""
    ctx = ctx or context()
    m, g = cfg.to_model()
    st = [np.ascontiguousarray(state[k], dtype=np.float64) for k in ("rates", "log_fx", "intens", "lagged")]
    if st[1].size == 0:
        st[1] = np.zeros(1)
    h = C.c_void_p()
    _lib.check(_lib.lib().hcva_simulate_conditional(
        ctx.handle, C.byref(m), C.byref(g), *[a.ctypes.data_as(_lib.dptr) for a in st], start_step,
        horizon, n_inner, stream.key, C.byref(h)))
    return SimulationSet(h, ctx)


def sample_default_block(sim: SimulationSet, n_replicas: int, stream: RandomStream) -> SimulationSet:
    """sample_default_block (defaults.cpp:20-45) on a simulated market, in place."""
    _lib.check(_lib.lib().hcva_sample_defaults(sim.handle, n_replicas, stream.key))
    sim.n_replicas = n_replicas
    return sim


def build_mtm_cube(sim: SimulationSet, book: np.ndarray) -> SimulationSet:
    """build_mtm_cube (portfolio.cpp:97-147) on a simulated market, in place."""
    bk, bp = _swaps(book)
    _lib.check(_lib.lib().hcva_build_cube(sim.handle, bp, len(bk)))
    return sim


def nested_cva(cfg: PipelineConfig, book: np.ndarray, states: Dict[str, np.ndarray], survived: np.ndarray,
               step: int, inner: int, parent: RandomStream, ctx: Optional[Context] = None, first_state: int = 0):
    """nested_cva (validation.cpp:123-179) for a batch of outer states.

    states: dict of arrays rates (S,E), log_fx (S,E-1), intens (S,Cn), lagged (S,E);
    survived: (S, Cc) bool; state s uses parent.split(first_state + s) (pipeline.cpp:284-288),
    so a rank holding states first_state.. of a larger set reproduces their estimates.
    Returns (value[S], std_error[S]).
    """
    ctx = ctx or context()
    m, g = cfg.to_model()
    S = states["rates"].shape[0]
    packed = np.ascontiguousarray(np.concatenate(
        [states["rates"], states["log_fx"].reshape(S, -1), states["intens"], states["lagged"]], axis=1),
        dtype=np.float64)
    surv = np.ascontiguousarray(survived, dtype=np.int32)
    bk, bp = _swaps(book)
    val, se = np.zeros(S), np.zeros(S)
    _lib.check(_lib.lib().hcva_nested_cva_range(
        ctx.handle, C.byref(m), C.byref(g), bp, len(bk), packed.ctypes.data_as(_lib.dptr),
        surv.ctypes.data_as(C.POINTER(C.c_int)), S, int(first_state), step, inner, parent.key,
        val.ctypes.data_as(_lib.dptr),
        se.ctypes.data_as(_lib.dptr)))
    return val, se


def twin_labels(sim: SimulationSet, book: np.ndarray, step: int, stream: RandomStream):
    """twin_labels (labels.cpp:90-140) of an outer set at `step`: (twin1, twin2), each (M, N).

    ``stream`` is the reference's twin stream (outer path k uses stream.split(k))."""
    bk, bp = _swaps(book)
    t1 = np.zeros((sim.n_paths, sim.n_replicas))
    t2 = np.zeros_like(t1)
    _lib.check(_lib.lib().hcva_twin_labels(sim.handle, bp, len(bk), int(step), stream.key,
                                           t1.ctypes.data_as(_lib.dptr), t2.ctypes.data_as(_lib.dptr)))
    return t1, t2


def _triplet(pred, t1, t2):
    out = [np.ascontiguousarray(np.ravel(a), dtype=np.float64) for a in (pred, t1, t2)]
    if not (out[0].size == out[1].size == out[2].size):
        raise _lib.ContractError("twin estimator: size mismatch or empty input")
    return out


def twin_l2_error(predictions, twin1, twin2, paths_per_block: int = 1):
    """twin_l2_error (validation.cpp:41-56): (value, clustered std error)."""
    p, a, b = _triplet(predictions, twin1, twin2)
    v, se = C.c_double(), C.c_double()
    _lib.check(_lib.lib().hcva_twin_l2_error(context().handle, p.ctypes.data_as(_lib.dptr), a.ctypes.data_as(_lib.dptr),
                                             b.ctypes.data_as(_lib.dptr), p.size, int(paths_per_block),
                                             C.byref(v), C.byref(se)))
    return v.value, se.value


def twin_relative_rmse(predictions, twin1, twin2) -> float:
    """twin_relative_rmse (validation.cpp:58-69); NumericError when E[xi1 xi2] <= 0."""
    p, a, b = _triplet(predictions, twin1, twin2)
    v = C.c_double()
    _lib.check(_lib.lib().hcva_twin_relative_rmse(context().handle, p.ctypes.data_as(_lib.dptr), a.ctypes.data_as(_lib.dptr),
                                                  b.ctypes.data_as(_lib.dptr), p.size, C.byref(v)))
    return v.value


def twin_relative_rmse_std_error(predictions, twin1, twin2, paths_per_block: int = 1) -> float:
    """twin_relative_rmse_std_error (validation.cpp:71-117)."""
    p, a, b = _triplet(predictions, twin1, twin2)
    v = C.c_double()
    _lib.check(_lib.lib().hcva_twin_relative_rmse_se(context().handle, p.ctypes.data_as(_lib.dptr), a.ctypes.data_as(_lib.dptr),
                                                     b.ctypes.data_as(_lib.dptr), p.size, int(paths_per_block),
                                                     C.byref(v)))
    return v.value


ARD_PRIOR = dict(vol_lo=0.5, vol_hi=1.5, level_lo=0.5, level_hi=2.0, speed_lo=0.5, speed_hi=1.5)  # ard.hpp:23-27


def ard_sample_variances(cfg: PipelineConfig, book: np.ndarray, n_dgp: int, paths_per_dgp: int,
                         stream: RandomStream, prior: Optional[Dict[str, float]] = None,
                         ctx: Optional[Context] = None) -> Dict[str, object]:
    """sample_variances (ard.cpp:56-125): per prior draw the time-averaged variances of the
    default indicators (v_x), market factors (v_y) and defaults labels (v_xi)."""
    ctx = ctx or context()
    m, g = cfg.to_model()
    pr = dict(ARD_PRIOR, **(prior or {}))
    pv = np.array([pr[k] for k in ("vol_lo", "vol_hi", "level_lo", "level_hi", "speed_lo", "speed_hi")])
    bk, bp = _swaps(book)
    C_, E = cfg.n_clients, cfg.n_economies
    vx, vy, vxi = np.zeros((n_dgp, C_)), np.zeros((n_dgp, 2 * E - 1 + C_)), np.zeros(n_dgp)
    rej = C.c_int()
    d = lambda a: a.ctypes.data_as(_lib.dptr)  # noqa: E731
    _lib.check(_lib.lib().hcva_ard_sample_variances(ctx.handle, C.byref(m), C.byref(g), bp, len(bk), d(pv), n_dgp,
                                                    paths_per_dgp, stream.key, d(vx), d(vy), d(vxi), C.byref(rej)))
    return dict(v_x=vx, v_y=vy, v_xi=vxi, rejected=rej.value)


def nested_relative_rmse(predictions: np.ndarray, nested: np.ndarray):
    """nested_relative_rmse (validation.cpp:181-210): (value, std_error, excluded_zero, used),
    reduced on the GPU (estimators.cu)."""
    pred = np.ascontiguousarray(np.ravel(predictions), dtype=np.float64)
    nest = np.ascontiguousarray(np.ravel(nested), dtype=np.float64)
    if pred.shape != nest.shape or pred.size == 0:
        raise _lib.ContractError("nested_relative_rmse: size mismatch or empty input")
    out = np.zeros(4)
    _lib.check(_lib.lib().hcva_nested_relative_rmse(context().handle, pred.ctypes.data_as(_lib.dptr),
                                                    nest.ctypes.data_as(_lib.dptr), pred.size,
                                                    out.ctypes.data_as(_lib.dptr)))
    return float(out[0]), float(out[1]), int(out[2]), int(out[3])


# ---- pybind-surface mirror (hiercva_module.cpp:99-139) ---------------------

def simulate(cfg: PipelineConfig, paths: int = 0, replicas: int = 0):
    """hiercva.simulate: (market, defaults, cube) from root.split(kTrainSim)."""
    book = resolve_book(cfg)
    sim = simulate_set(cfg, book, paths if paths > 0 else cfg.paths,
                       replicas if replicas > 0 else cfg.replicas,
                       RandomStream(cfg.seed).split(K_TRAIN_SIM))
    sim.book = book
    return sim, sim, sim


def _ensure_cube(cfg: PipelineConfig, sim: SimulationSet) -> None:
    if getattr(sim, "book", None) is None:
        sim.book = resolve_book(cfg)
        build_mtm_cube(sim, sim.book)


def defaults_label(step: int, cfg: PipelineConfig, market: SimulationSet, defaults=None) -> np.ndarray:
    _ensure_cube(cfg, market)
    return market.labels(step, "defaults")


def intensity_label(step: int, cfg: PipelineConfig, market: SimulationSet, defaults=None) -> np.ndarray:
    _ensure_cube(cfg, market)
    return market.labels(step, "intensity")


def features(step: int, market: SimulationSet, defaults=None) -> np.ndarray:
    return market.features(step)
