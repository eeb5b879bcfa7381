"""ctypes declarations of libhcva_gpu.so (include/hcva_gpu.h).

The product path is this library and nothing else: when the shared object is
missing or no B200 is visible the calls raise -- there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("HCVA_LIB") or os.path.join(PKG, "lib", "libhcva_gpu.so")
CSRC = os.path.join(PKG, "csrc")

u64 = C.c_uint64
dptr = C.POINTER(C.c_double)


class Vasicek(C.Structure):
    _fields_ = [("a", C.c_double), ("b", C.c_double), ("sigma", C.c_double), ("r0", C.c_double)]


class Fx(C.Structure):
    _fields_ = [("sigma", C.c_double), ("rho", C.c_double), ("chi0", C.c_double)]


class Cir(C.Structure):
    _fields_ = [("alpha", C.c_double), ("delta", C.c_double), ("nu", C.c_double), ("gamma0", C.c_double)]


class Model(C.Structure):
    _fields_ = [("n_economies", C.c_int), ("n_clients", C.c_int), ("rates", C.POINTER(Vasicek)),
                ("fx", C.POINTER(Fx)), ("credit", C.POINTER(Cir)), ("correlation", dptr)]


class Grid(C.Structure):
    _fields_ = [("n_steps", C.c_int), ("substeps", C.c_int), ("dt", C.c_double)]


class Swap(C.Structure):
    _fields_ = [("economy", C.c_int), ("client", C.c_int), ("notional", C.c_double),
                ("tenor", C.c_double), ("maturity", C.c_double), ("fixed_rate", C.c_double)]


class TrainCfg(C.Structure):
    _fields_ = [("epochs", C.c_int), ("n_batches", C.c_int), ("hidden_layers", C.c_int), ("width", C.c_int),
                ("activation", C.c_int), ("adam", C.c_int), ("learning_rate", C.c_double), ("ridge", C.c_double),
                ("seed", u64)]


# Status codes (include/hcva_gpu.h) -> exception types of the reference
# (proj/include/hiercva/errors.hpp:9-25, hiercva_module.cpp:49-50).
class HcvaError(RuntimeError):
    pass


class ConfigError(HcvaError):
    pass


class ContractError(HcvaError):
    pass


class NumericError(HcvaError):
    pass


class CudaError(HcvaError):
    pass


_ERRORS = {1: ConfigError, 2: ContractError, 3: NumericError, 4: CudaError}


def build(force: bool = False) -> str:
    """Compile libhcva_gpu.so in-tree for sm_100a (nvcc cross-compiles on CPU)."""
    if force or not os.path.exists(LIB_PATH):
        subprocess.run(["make", "-s", "-C", CSRC], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CudaError(f"{LIB_PATH} is not built; run paper_2211_17005_b200._lib.build() "
                        "(the engine has no CPU fallback)")
    L = C.CDLL(LIB_PATH)
    st = C.c_int
    vp = C.c_void_p
    L.hcva_last_error.restype = C.c_char_p
    L.hcva_version.restype = C.c_char_p
    L.hcva_rng_root_key.restype = u64
    L.hcva_rng_root_key.argtypes = [u64]
    L.hcva_rng_split_key.restype = u64
    L.hcva_rng_split_key.argtypes = [u64, u64]
    sigs = {
        "hcva_ctx_create": [C.c_int, C.POINTER(vp)],
        "hcva_ctx_destroy": [vp],
        "hcva_ctx_stream": [vp, C.POINTER(vp)],
        "hcva_ctx_synchronize": [vp],
        "hcva_ctx_launch_count": [vp, C.POINTER(u64)],
        "hcva_rng_draw": [vp, u64, u64, C.c_size_t, C.c_int, vp],
        "hcva_cholesky": [C.POINTER(Model), dptr],
        "hcva_par_rate": [C.c_double, C.c_double, C.POINTER(Vasicek), dptr],
        "hcva_zc_price": [C.c_double, C.c_double, C.POINTER(Vasicek), dptr],
        "hcva_generate_book": [C.POINTER(Model), C.POINTER(Grid), C.c_int, C.c_double, C.c_double,
                               u64, C.POINTER(Swap)],
        "hcva_simulate_set": [vp, C.POINTER(Model), C.POINTER(Grid), C.POINTER(Swap), C.c_int,
                              C.c_int, C.c_int, C.c_int, u64, u64, C.POINTER(vp)],
        "hcva_simulate_set_sharded": [vp, C.POINTER(Model), C.POINTER(Grid), C.POINTER(Swap), C.c_int,
                                      C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, u64, u64, C.POINTER(vp)],
        "hcva_simulate_conditional": [vp, C.POINTER(Model), C.POINTER(Grid), dptr, dptr, dptr, dptr,
                                      C.c_int, C.c_int, C.c_int, u64, C.POINTER(vp)],
        "hcva_sample_defaults": [vp, C.c_int, u64],
        "hcva_build_cube": [vp, C.POINTER(Swap), C.c_int],
        "hcva_sim_destroy": [vp],
        "hcva_sim_dims": [vp, C.POINTER(C.c_int)],
        "hcva_sim_tie_counts": [vp, C.POINTER(u64)],
        "hcva_sim_export_market": [vp, vp, vp, vp, vp, vp, vp],
        "hcva_sim_export_defaults": [vp, vp],
        "hcva_sim_export_cube": [vp, vp],
        "hcva_labels": [vp, C.c_int, C.c_int, vp],
        "hcva_labels_all": [vp, C.c_int, vp],
        "hcva_features": [vp, C.c_int, vp],
        "hcva_sim_rerun": [vp, u64, u64, C.c_int, C.c_int],
        "hcva_sim_phase_times": [vp, C.c_int, C.POINTER(C.c_float)],
        "hcva_cva_profile": [vp, C.c_int, vp],
        "hcva_diag_fp64_peak": [vp, dptr],
        "hcva_diag_special": [vp, C.c_int, vp, C.c_size_t, vp],
        "hcva_diag_tc_gemm": [vp, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp],
        "hcva_diag_tc_rate": [vp, C.c_int, C.c_int, C.c_int, dptr],
        "hcva_nested_cva_batch": [vp, C.POINTER(Model), C.POINTER(Grid), C.POINTER(Swap), C.c_int, dptr,
                                  C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, u64, dptr, dptr],
        "hcva_nested_cva_range": [vp, C.POINTER(Model), C.POINTER(Grid), C.POINTER(Swap), C.c_int, dptr,
                                  C.POINTER(C.c_int), C.c_int, C.c_int, C.c_int, C.c_int, u64, dptr, dptr],
        "hcva_net_size": [C.POINTER(TrainCfg), C.c_int, C.POINTER(C.c_int)],
        "hcva_init_network": [C.POINTER(TrainCfg), C.c_int, u64, dptr],
        "hcva_quadratic_loss": [vp, C.POINTER(TrainCfg), C.c_int, dptr, C.c_int, dptr, dptr, C.c_int, dptr, dptr],
        "hcva_forward": [vp, C.POINTER(TrainCfg), C.c_int, dptr, dptr, C.c_int, dptr],
        "hcva_refit_output_layer": [vp, C.POINTER(TrainCfg), C.c_int, dptr, dptr, dptr, C.c_int],
        "hcva_diag_sgd_timing": [vp, C.POINTER(TrainCfg), C.c_int, C.c_int, C.c_int, dptr],
        "hcva_sim_quadratic_loss": [vp, C.POINTER(TrainCfg), C.c_int, C.c_int, dptr, dptr, dptr, C.c_int, C.c_long,
                                    C.c_long, dptr, dptr],
        "hcva_train_base": [vp, C.POINTER(TrainCfg), C.c_int, dptr, dptr, C.c_int, dptr, dptr, dptr, dptr,
                            C.POINTER(C.c_int)],
        "hcva_backward_learn": [vp, C.POINTER(TrainCfg), C.c_int, C.POINTER(vp)],
        "hcva_backward_learn_dist": [vp, C.POINTER(TrainCfg), C.c_int, vp, C.POINTER(vp)],
        "hcva_twin_labels": [vp, C.POINTER(Swap), C.c_int, C.c_int, u64, dptr, dptr],
        "hcva_backward_learn_qr": [vp, C.POINTER(TrainCfg), C.c_int, u64, dptr, C.POINTER(vp)],
        "hcva_probe_block": [vp, u64, C.c_int, C.POINTER(C.c_uint16), dptr],
        "hcva_estimate_qr": [vp, dptr, dptr, C.c_size_t, dptr],
        "hcva_nested_relative_rmse": [vp, dptr, dptr, C.c_size_t, dptr],
        "hcva_percentile_table": [vp, vp, dptr],
        "hcva_ard_sample_variances": [vp, C.POINTER(Model), C.POINTER(Grid), C.POINTER(Swap), C.c_int, dptr,
                                      C.c_int, C.c_int, u64, dptr, dptr, dptr, C.POINTER(C.c_int)],
        "hcva_models_save": [vp, C.c_char_p, u64, C.c_char_p],
        "hcva_models_load": [vp, C.c_char_p, C.POINTER(u64), C.c_char_p, C.c_int, C.POINTER(vp)],
        "hcva_sim_save_market": [vp, C.c_char_p, u64],
        "hcva_market_load": [vp, C.POINTER(Model), C.POINTER(Grid), C.c_char_p, C.POINTER(u64), C.POINTER(vp)],
        "hcva_twin_l2_error": [vp, dptr, dptr, dptr, C.c_size_t, C.c_int, dptr, dptr],
        "hcva_twin_relative_rmse": [vp, dptr, dptr, dptr, C.c_size_t, dptr],
        "hcva_twin_relative_rmse_se": [vp, dptr, dptr, dptr, C.c_size_t, C.c_int, dptr],
        "hcva_comm_nccl_id": [C.c_char_p],
        "hcva_comm_create_nccl": [vp, C.c_int, C.c_int, C.c_char_p, C.POINTER(vp)],
        "hcva_group_create": [C.c_int, C.POINTER(vp)],
        "hcva_group_destroy": [vp],
        "hcva_comm_create_local": [vp, vp, C.c_int, C.POINTER(vp)],
        "hcva_comm_info": [vp, C.POINTER(C.c_int), C.POINTER(C.c_int)],
        "hcva_comm_destroy": [vp],
        "hcva_models_info": [vp, C.POINTER(C.c_int)],
        "hcva_models_get": [vp, C.c_int, dptr, dptr, dptr, dptr, dptr, C.POINTER(C.c_int)],
        "hcva_predict": [vp, vp, C.c_int, dptr],
        "hcva_models_destroy": [vp],
    }
    for name, args in sigs.items():
        fn = getattr(L, name)
        fn.argtypes = args
        fn.restype = st
    _lib = L
    return L


def check(rc: int) -> None:
    if rc != 0:
        msg = lib().hcva_last_error().decode()
        raise _ERRORS.get(rc, HcvaError)(msg)


# Every symbol include/hcva_gpu.h declares (checked by tests/test_abi.py).
EXPORTED = [
    "hcva_last_error", "hcva_version", "hcva_ctx_create", "hcva_ctx_destroy", "hcva_ctx_stream",
    "hcva_ctx_synchronize", "hcva_ctx_launch_count", "hcva_rng_root_key", "hcva_rng_split_key",
    "hcva_rng_draw", "hcva_cholesky", "hcva_par_rate", "hcva_zc_price", "hcva_generate_book",
    "hcva_simulate_set", "hcva_simulate_set_sharded", "hcva_simulate_conditional", "hcva_sample_defaults", "hcva_build_cube",
    "hcva_sim_destroy", "hcva_sim_dims", "hcva_sim_tie_counts", "hcva_sim_export_market",
    "hcva_sim_export_defaults", "hcva_sim_export_cube", "hcva_labels", "hcva_labels_all",
    "hcva_features", "hcva_sim_rerun", "hcva_sim_phase_times", "hcva_cva_profile",
    "hcva_diag_fp64_peak", "hcva_diag_special", "hcva_diag_tc_gemm", "hcva_diag_tc_rate", "hcva_nested_cva_batch", "hcva_nested_cva_range", "hcva_net_size",
    "hcva_init_network", "hcva_quadratic_loss", "hcva_train_base", "hcva_backward_learn", "hcva_models_info",
    "hcva_models_get", "hcva_predict", "hcva_models_destroy", "hcva_comm_nccl_id", "hcva_comm_create_nccl",
    "hcva_group_create", "hcva_group_destroy", "hcva_comm_create_local", "hcva_comm_info", "hcva_comm_destroy",
    "hcva_backward_learn_dist", "hcva_twin_labels", "hcva_twin_l2_error", "hcva_twin_relative_rmse",
    "hcva_twin_relative_rmse_se", "hcva_backward_learn_qr", "hcva_probe_block", "hcva_estimate_qr",
    "hcva_models_save", "hcva_models_load", "hcva_sim_save_market", "hcva_market_load",
    "hcva_ard_sample_variances", "hcva_nested_relative_rmse", "hcva_percentile_table",
    "hcva_forward", "hcva_refit_output_layer", "hcva_diag_sgd_timing", "hcva_sim_quadratic_loss",
]
