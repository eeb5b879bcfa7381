"""B200-native pathwise CVA engine (arXiv 2211.17005), drop-in for the hot path
of the reference `hiercva` library.  See DESIGN.md / INTEGRATION.md.

The compute path is libhcva_gpu.so (hand-written sm_100a CUDA behind the C ABI
in include/hcva_gpu.h); this package is its host-side mirror of the
reference's pybind surface (proj/python/hiercva/__init__.py:14-35).
"""
from ._lib import ConfigError, ContractError, CudaError, HcvaError, NumericError, build  # noqa: F401
from .config import PipelineConfig, TrainConfig, load_config, parse_config  # noqa: F401
from .engine import (  # noqa: F401
    K_BOOK, K_TRAIN_SIM, K_VALIDATION_SIM, SWAP_DTYPE, Context, RandomStream, SimulationSet,
    build_mtm_cube, cholesky, context, defaults_label, features, generate_book, intensity_label,
    load_book_csv, nested_cva, nested_relative_rmse, twin_l2_error, twin_labels, twin_relative_rmse,
    twin_relative_rmse_std_error, load_market, save_book_csv, ard_sample_variances, par_rate, resolve_book, sample_default_block, simulate, simulate_conditional_market,
    simulate_market, simulate_set, zc_price,
)

__all__ = [
    "twin_labels", "twin_l2_error", "twin_relative_rmse", "twin_relative_rmse_std_error",
    "ConfigError", "NumericError", "ContractError", "CudaError", "PipelineConfig", "RandomStream",
    "SimulationSet", "defaults_label", "features", "intensity_label", "load_config", "parse_config",
    "simulate", "simulate_set", "simulate_market", "simulate_conditional_market",
    "sample_default_block", "build_mtm_cube", "generate_book", "resolve_book", "par_rate", "zc_price",
]
