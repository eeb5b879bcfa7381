"""ctypes bindings for the CPU oracle libraries -- TEST INFRASTRUCTURE ONLY.

Loads either the plain-C restatement (oracle/liboracle.so) or the compiled
reference (oracle/_ref/libhcva_ref.so); both export the C interface declared in
oracle/hcva_oracle.h.  Used only by tests/, __graft_entry__.smoke() and the
cpu_baseline / --impl reference legs of bench.py.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_DIR = os.path.join(ROOT, "oracle")
RESTATEMENT = os.path.join(ORACLE_DIR, "liboracle.so")
REFERENCE = os.path.join(ORACLE_DIR, "_ref", "libhcva_ref.so")

_u64 = C.c_uint64
_dp = C.POINTER(C.c_double)


class OrModel(C.Structure):
    _fields_ = [
        ("n_economies", C.c_int),
        ("n_clients", C.c_int),
        ("rates", _dp),
        ("fx", _dp),
        ("credit", _dp),
        ("corr", _dp),
        ("n_steps", C.c_int),
        ("substeps", C.c_int),
        ("dt", C.c_double),
    ]


SWAP_DTYPE = np.dtype(
    [("economy", "<i4"), ("client", "<i4"), ("notional", "<f8"), ("tenor", "<f8"),
     ("maturity", "<f8"), ("fixed_rate", "<f8")],
    align=True,
)


def build():
    """Compile the restatement (and, where /root/reference exists, the reference)."""
    subprocess.run(["make", "-s", "-C", ORACLE_DIR], check=True)


def _ptr(a, ctype=C.c_double):
    return a.ctypes.data_as(C.POINTER(ctype))


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class Oracle:
    """One oracle library (restatement or compiled reference)."""

    def __init__(self, path=RESTATEMENT):
        if not os.path.exists(path):
            build()
        self.path = path
        self.lib = C.CDLL(path)
        L = self.lib
        L.or_last_error.restype = C.c_char_p
        L.or_root_key.restype = _u64
        L.or_root_key.argtypes = [_u64]
        L.or_split_key.restype = _u64
        L.or_split_key.argtypes = [_u64, _u64]
        for name in ("or_uniforms", "or_normals", "or_exponentials"):
            getattr(L, name).argtypes = [_u64, _u64, C.c_size_t, _dp]
        L.or_draw_u64.argtypes = [_u64, _u64, C.c_size_t, C.POINTER(_u64)]
        L.or_inverse_normal_cdf.restype = C.c_double
        L.or_inverse_normal_cdf.argtypes = [C.c_double]
        self._keep = []

    # -- helpers ---------------------------------------------------------
    def _check(self, rc):
        if rc != 0:
            raise OracleError(rc, self.lib.or_last_error().decode())

    def model(self, m):
        """m: dict with rates (E,4), fx (E-1,3), credit (Cc+1,4), corr or None, grid."""
        rates = np.ascontiguousarray(m["rates"], dtype=np.float64)
        fx = np.ascontiguousarray(m["fx"], dtype=np.float64).reshape(-1)
        if fx.size == 0:
            fx = np.zeros(1)
        credit = np.ascontiguousarray(m["credit"], dtype=np.float64)
        corr = m.get("corr")
        corr = None if corr is None else np.ascontiguousarray(corr, dtype=np.float64)
        self._keep = [rates, fx, credit, corr]
        return OrModel(rates.shape[0], credit.shape[0] - 1, _ptr(rates), _ptr(fx), _ptr(credit),
                       _ptr(corr) if corr is not None else _dp(), m["n_steps"], m["substeps"],
                       m["dt"])

    # -- RNG -------------------------------------------------------------
    def key(self, seed, *lineage):
        k = self.lib.or_root_key(seed)
        for x in lineage:
            k = self.lib.or_split_key(k, x)
        return k

    def split(self, key, k):
        return self.lib.or_split_key(key, k)

    def u64(self, key, start, count):
        out = np.zeros(count, dtype=np.uint64)
        self.lib.or_draw_u64(key, start, count, _ptr(out, _u64))
        return out

    def uniforms(self, key, start, count):
        out = np.zeros(count)
        self.lib.or_uniforms(key, start, count, _ptr(out))
        return out

    def normals(self, key, start, count):
        out = np.zeros(count)
        self.lib.or_normals(key, start, count, _ptr(out))
        return out

    def exponentials(self, key, start, count):
        out = np.zeros(count)
        self.lib.or_exponentials(key, start, count, _ptr(out))
        return out

    # -- simulation ------------------------------------------------------
    def simulate_market(self, m, n_paths, key):
        E, Cn, n = len(m["rates"]), len(m["credit"]), m["n_steps"]
        rows = n_paths * (n + 1)
        out = dict(rates=np.zeros((n_paths, n + 1, E)), fx=np.zeros((n_paths, n + 1, max(E - 1, 0))),
                   intens=np.zeros((n_paths, n + 1, Cn)), lagged=np.zeros((n_paths, n + 1, E)),
                   disc=np.zeros((n_paths, n + 1)), hazard=np.zeros((n_paths, n + 1, Cn)))
        fxbuf = out["fx"] if E > 1 else np.zeros(rows)
        mm = self.model(m)
        self._check(self.lib.or_simulate_market(
            C.byref(mm), n_paths, _u64(key), _ptr(out["rates"]), _ptr(fxbuf), _ptr(out["intens"]),
            _ptr(out["lagged"]), _ptr(out["disc"]), _ptr(out["hazard"])))
        return out

    def simulate_conditional(self, m, state, start_step, horizon, n_inner, key):
        E, Cn = len(m["rates"]), len(m["credit"])
        rows = n_inner * (horizon + 1)
        out = dict(rates=np.zeros((n_inner, horizon + 1, E)),
                   fx=np.zeros((n_inner, horizon + 1, max(E - 1, 0))),
                   intens=np.zeros((n_inner, horizon + 1, Cn)),
                   lagged=np.zeros((n_inner, horizon + 1, E)), disc=np.zeros((n_inner, horizon + 1)),
                   hazard=np.zeros((n_inner, horizon + 1, Cn)))
        fxbuf = out["fx"] if E > 1 else np.zeros(rows)
        st = [np.ascontiguousarray(state[k], dtype=np.float64)
              for k in ("rates", "log_fx", "intens", "lagged")]
        if st[1].size == 0:
            st[1] = np.zeros(1)
        mm = self.model(m)
        self._check(self.lib.or_simulate_conditional(
            C.byref(mm), _ptr(st[0]), _ptr(st[1]), _ptr(st[2]), _ptr(st[3]), start_step, horizon,
            n_inner, _u64(key), _ptr(out["rates"]), _ptr(fxbuf), _ptr(out["intens"]),
            _ptr(out["lagged"]), _ptr(out["disc"]), _ptr(out["hazard"])))
        return out

    def sample_defaults(self, hazard, n_replicas, key):
        M, n1, Cn = hazard.shape
        hz = np.ascontiguousarray(hazard)
        out = np.zeros((M, n_replicas, Cn), dtype=np.uint16)
        self._check(self.lib.or_sample_defaults(M, n1 - 1, Cn, _ptr(hz), n_replicas, _u64(key),
                                                _ptr(out, C.c_uint16)))
        return out

    def zc_price(self, r, tau, v):
        v = np.asarray(v, dtype=np.float64)
        out = C.c_double()
        self._check(self.lib.or_zc_price(C.c_double(r), C.c_double(tau), _ptr(v), C.byref(out)))
        return out.value

    def par_rate(self, maturity, tenor, v):
        v = np.asarray(v, dtype=np.float64)
        out = C.c_double()
        self._check(self.lib.or_par_rate(C.c_double(maturity), C.c_double(tenor), _ptr(v),
                                         C.byref(out)))
        return out.value

    def generate_book(self, m, count, nmin, nmax, key):
        out = np.zeros(count, dtype=SWAP_DTYPE)
        mm = self.model(m)
        self._check(self.lib.or_generate_book(C.byref(mm), count, C.c_double(nmin),
                                              C.c_double(nmax), _u64(key), out.ctypes.data_as(C.c_void_p)))
        return out

    def build_cube(self, m, market, book, start_step=0):
        rates = np.ascontiguousarray(market["rates"])
        M, n1, E = rates.shape
        fx = np.ascontiguousarray(market["fx"]) if E > 1 else np.zeros(M * n1)
        lagged = np.ascontiguousarray(market["lagged"])
        Cc = len(m["credit"]) - 1
        cube = np.zeros((M, n1, Cc))
        book = np.ascontiguousarray(book, dtype=SWAP_DTYPE)
        mm = self.model(m)
        self._check(self.lib.or_build_cube(C.byref(mm), M, n1 - 1, start_step, _ptr(rates),
                                           _ptr(fx), _ptr(lagged), book.ctypes.data_as(C.c_void_p),
                                           len(book), _ptr(cube)))
        return cube

    def _label(self, fn, step, market, steps, cube, dt):
        disc = np.ascontiguousarray(market["disc"])
        intens = np.ascontiguousarray(market["intens"])
        M, n1 = disc.shape
        E = market["rates"].shape[2]
        Cn = intens.shape[2]
        N = steps.shape[1]
        out = np.zeros((M, N))
        st = np.ascontiguousarray(steps, dtype=np.uint16)
        cb = np.ascontiguousarray(cube)
        self._check(fn(int(step), M, n1 - 1, E, Cn, N, C.c_double(dt), _ptr(disc), _ptr(intens),
                       _ptr(st, C.c_uint16), _ptr(cb), _ptr(out)))
        return out

    def defaults_label(self, step, market, steps, cube, dt):
        return self._label(self.lib.or_defaults_label, step, market, steps, cube, dt)

    def intensity_label(self, step, market, steps, cube, dt):
        return self._label(self.lib.or_intensity_label, step, market, steps, cube, dt)

    def features(self, step, market, steps):
        rates = np.ascontiguousarray(market["rates"])
        M, n1, E = rates.shape
        fx = np.ascontiguousarray(market["fx"]) if E > 1 else np.zeros(M * n1)
        intens = np.ascontiguousarray(market["intens"])
        lagged = np.ascontiguousarray(market["lagged"])
        Cn = intens.shape[2]
        N = steps.shape[1]
        cols = (Cn - 1) + E + (E - 1) + (Cn - 1) + E
        out = np.zeros((M * N, cols))
        st = np.ascontiguousarray(steps, dtype=np.uint16)
        self._check(self.lib.or_features(int(step), M, n1 - 1, E, Cn, N, _ptr(rates), _ptr(fx),
                                         _ptr(intens), _ptr(lagged), _ptr(st, C.c_uint16),
                                         _ptr(out)))
        return out

    def nested_cva(self, m, book, state, survived, step, inner, key):
        st = [np.ascontiguousarray(state[k], dtype=np.float64)
              for k in ("rates", "log_fx", "intens", "lagged")]
        if st[1].size == 0:
            st[1] = np.zeros(1)
        surv = np.ascontiguousarray(survived, dtype=np.int32)
        book = np.ascontiguousarray(book, dtype=SWAP_DTYPE)
        v, se = C.c_double(), C.c_double()
        mm = self.model(m)
        self._check(self.lib.or_nested_cva(C.byref(mm), book.ctypes.data_as(C.c_void_p), len(book),
                                           _ptr(st[0]), _ptr(st[1]), _ptr(st[2]), _ptr(st[3]),
                                           _ptr(surv, C.c_int), int(step), int(inner), _u64(key),
                                           C.byref(v), C.byref(se)))
        return v.value, se.value


    # -- twin MC validator (labels.cpp:90-140, validation.cpp:41-117) -------
    def twin_labels(self, m, book, step, market, steps, key):
        rates = np.ascontiguousarray(market["rates"])
        M, n1, E = rates.shape
        fx = np.ascontiguousarray(market["fx"]) if E > 1 else np.zeros(M * n1)
        intens = np.ascontiguousarray(market["intens"])
        lagged = np.ascontiguousarray(market["lagged"])
        st = np.ascontiguousarray(steps, dtype=np.uint16)
        N = st.shape[1]
        t1, t2 = np.zeros((M, N)), np.zeros((M, N))
        book = np.ascontiguousarray(book, dtype=SWAP_DTYPE)
        mm = self.model(m)
        self._check(self.lib.or_twin_labels(C.byref(mm), book.ctypes.data_as(C.c_void_p), len(book), int(step), M, N,
                                            _ptr(rates), _ptr(fx), _ptr(intens), _ptr(lagged),
                                            _ptr(st, C.c_uint16), _u64(key), _ptr(t1), _ptr(t2)))
        return t1, t2

    def _triplet(self, pred, t1, t2):
        return [np.ascontiguousarray(np.ravel(a), dtype=np.float64) for a in (pred, t1, t2)]

    def twin_l2_error(self, pred, t1, t2, block=1):
        p, a, b = self._triplet(pred, t1, t2)
        v, se = C.c_double(), C.c_double()
        self._check(self.lib.or_twin_l2_error(_ptr(p), _ptr(a), _ptr(b), C.c_size_t(p.size), int(block),
                                              C.byref(v), C.byref(se)))
        return v.value, se.value

    def twin_relative_rmse(self, pred, t1, t2):
        p, a, b = self._triplet(pred, t1, t2)
        v = C.c_double()
        self._check(self.lib.or_twin_relative_rmse(_ptr(p), _ptr(a), _ptr(b), C.c_size_t(p.size), C.byref(v)))
        return v.value

    def twin_relative_rmse_std_error(self, pred, t1, t2, block=1):
        p, a, b = self._triplet(pred, t1, t2)
        v = C.c_double()
        self._check(self.lib.or_twin_relative_rmse_se(_ptr(p), _ptr(a), _ptr(b), C.c_size_t(p.size), int(block),
                                                      C.byref(v)))
        return v.value

    def ard_sample_variances(self, m, book, prior, n_dgp, paths, key):
        C_ = len(m["credit"]) - 1
        E = len(m["rates"])
        vx, vy, vxi = np.zeros((n_dgp, C_)), np.zeros((n_dgp, 2 * E - 1 + C_)), np.zeros(n_dgp)
        rej = C.c_int()
        pv = np.ascontiguousarray(prior, dtype=np.float64)
        book = np.ascontiguousarray(book, dtype=SWAP_DTYPE)
        mm = self.model(m)
        self._check(self.lib.or_ard_sample_variances(C.byref(mm), book.ctypes.data_as(C.c_void_p), len(book),
                                                     _ptr(pv), n_dgp, paths, _u64(key), _ptr(vx), _ptr(vy),
                                                     _ptr(vxi), C.byref(rej)))
        return dict(v_x=vx, v_y=vy, v_xi=vxi, rejected=rej.value)

    def estimate_qr(self, g1, g2):
        """planner.cpp:11-70 -> dict(q, r, total, n_pairs, q_std_error, r_std_error)."""
        a = np.ascontiguousarray(g1, dtype=np.float64)
        b = np.ascontiguousarray(g2, dtype=np.float64)
        out = np.zeros(6)
        self._check(self.lib.or_estimate_qr(_ptr(a), _ptr(b), C.c_size_t(a.size), _ptr(out)))
        return dict(q=out[0], r=out[1], total=out[2], n_pairs=int(out[3]), q_std_error=out[4], r_std_error=out[5])

    def nested_relative_rmse(self, pred, nested):
        """validation.cpp:181-210 -> (value, std_error, excluded_zero, used)."""
        p = np.ascontiguousarray(np.ravel(pred), dtype=np.float64)
        v = np.ascontiguousarray(np.ravel(nested), dtype=np.float64)
        out = np.zeros(4)
        self._check(self.lib.or_nested_relative_rmse(_ptr(p), _ptr(v), C.c_size_t(p.size), _ptr(out)))
        return float(out[0]), float(out[1]), int(out[2]), int(out[3])

    def percentile_bands(self, values):
        """One percentile_table row (pipeline.cpp:41-47,138-156): mean, p1, p2.5, p97.5, p99."""
        v = np.array(np.ravel(values), dtype=np.float64)
        out = np.zeros(5)
        self._check(self.lib.or_percentile_bands(_ptr(v), C.c_size_t(v.size), _ptr(out)))
        return out

    # -- regression (regressor.cpp restated) -------------------------------
    def _shape(self, d, hidden, width, activation=0):
        class S(C.Structure):
            _fields_ = [("input_dim", C.c_int), ("hidden", C.c_int), ("width", C.c_int), ("activation", C.c_int)]
        return S(d, hidden, width, activation)

    def net_size(self, d, hidden, width):
        self.lib.or_net_size.restype = C.c_size_t
        return self.lib.or_net_size(C.byref(self._shape(d, hidden, width)))

    def init_network(self, d, hidden, width, key):
        p = np.zeros(self.net_size(d, hidden, width))
        self.lib.or_init_network(C.byref(self._shape(d, hidden, width)), _u64(key), _ptr(p))
        return p

    def fit_scaler(self, x, passthrough):
        x = np.ascontiguousarray(x, dtype=np.float64)
        mean, scale = np.zeros(x.shape[1]), np.zeros(x.shape[1])
        self.lib.or_fit_scaler(_ptr(x), x.shape[0], x.shape[1], passthrough, _ptr(mean), _ptr(scale))
        return mean, scale

    def forward(self, p, x, hidden, width, activation=0, head=True):
        x = np.ascontiguousarray(x, dtype=np.float64)
        p = np.ascontiguousarray(p, dtype=np.float64)
        out = np.zeros(x.shape[0])
        self.lib.or_forward(C.byref(self._shape(x.shape[1], hidden, width, activation)), _ptr(p), int(head),
                            _ptr(x), x.shape[0], _ptr(out))
        return out

    def loss(self, p, x, y, hidden, width, activation=0, head=False, grads=True):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        p = np.ascontiguousarray(p, dtype=np.float64)
        g = np.zeros_like(p) if grads else None
        self.lib.or_quadratic_loss.restype = C.c_double
        v = self.lib.or_quadratic_loss(C.byref(self._shape(x.shape[1], hidden, width, activation)), _ptr(p),
                                       int(head), _ptr(x), _ptr(y), x.shape[0], _ptr(g) if grads else _dp())
        return (v, g) if grads else v

    def refit(self, p, x, y, hidden, width, ridge=1e-8, activation=0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        p = np.array(p, dtype=np.float64)
        self.lib.or_refit(C.byref(self._shape(x.shape[1], hidden, width, activation)), _ptr(p), _ptr(x), _ptr(y),
                          x.shape[0], C.c_double(ridge))
        return p

    def train_base(self, x, y, init, hidden, width, n_batches, epochs, lr=1e-3, adam=True, ridge=1e-8,
                   activation=0):
        x = np.ascontiguousarray(x, dtype=np.float64)
        y = np.ascontiguousarray(y, dtype=np.float64)
        init = np.ascontiguousarray(init, dtype=np.float64)
        best = np.zeros_like(init)
        losses = np.zeros(epochs)
        bl, be = C.c_double(), C.c_int()
        self._check(self.lib.or_train_base(
            C.byref(self._shape(x.shape[1], hidden, width, activation)), _ptr(x), _ptr(y), x.shape[0], n_batches,
            epochs, C.c_double(lr), int(adam), C.c_double(ridge), _ptr(init), _ptr(best), _ptr(losses),
            C.byref(bl), C.byref(be)))
        return best, dict(epoch_losses=losses, best_loss=bl.value, best_epoch=be.value)

    def backward_learn(self, n_steps, source, seed, hidden, width, n_batches, epochs, lr=1e-3, adam=True,
                       ridge=1e-8, activation=0):
        """regressor.cpp:354-395 (Alg. 2): i = n..1, fit_scaler, init at n (mu = label mean)
        else warm start from step i+1's best; returns {i: (params, mean, scale, report)}."""
        out, carry = {}, None
        for i in range(n_steps, 0, -1):
            x, y, passthrough = source(i)
            mean, scale = self.fit_scaler(x, passthrough)
            xs = (x - mean) / scale
            if i == n_steps:
                start = self.init_network(x.shape[1], hidden, width, self.key(seed, 0xBEEF, i))
                start[-1] = float(np.mean(y))
            else:
                start = carry
            best, rep = self.train_base(xs, y, start, hidden, width, n_batches, epochs, lr, adam, ridge, activation)
            carry = best
            out[i] = (best, mean, scale, rep)
        return out


_cache = {}


def restatement():
    if "r" not in _cache:
        _cache["r"] = Oracle(RESTATEMENT)
    return _cache["r"]


def reference():
    """The compiled reference, or None where /root/reference was never built."""
    if "ref" not in _cache:
        if not os.path.exists(REFERENCE):
            try:
                build()
            except Exception:
                pass
        _cache["ref"] = Oracle(REFERENCE) if os.path.exists(REFERENCE) else None
    return _cache["ref"]
