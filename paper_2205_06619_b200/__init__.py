"""B200-native FastSTMF (arXiv 2205.06619): a drop-in for the reference package's
fitting path (``tropfact.fast_stmf`` / ``tropfact.fit``) running on sm_100a.

Host code (this package) keeps the reference's API and its numpy RNG draws
(orientation, Random-Acol picks); every fit computation runs in the CUDA library
``lib/libstmf_b200.so`` (C ABI in include/stmf_b200.h).  No CPU fallback.
"""

from .types import (FactorPair, MaskedMatrix, Orientation, Permutation, RunConfig, Trajectory,
                    UpdateOutcome)
from .engine import FitSession, f_ulf, f_urf, random_acol_init, run_fit, stmf_baseline
from .strategies import BASELINE, FASTSTMF, StrategySpec, fast_stmf, fit, parse_method
from .tropical import (approx_error, argmax_grid, argmax_k, b_norm, masked_minplus, sort_perm_by_min, td, td_col,
                       td_grid, td_row, trop_matmul)
from ._ext import build, StmfError
from . import datagen, io, metrics
from .datagen import SynthSpec, apply_mask, gen_mixture, gen_tall_wide_pair
from .metrics import (NEVER, bootstrap_ci, distance_correlation, masked_dc, nemenyi_cd, normalized_error, omega,
                      rank_methods, rmse, time_to_reach)

__version__ = "0.1.0"

__all__ = [
    "MaskedMatrix", "Permutation", "trop_matmul", "masked_minplus", "approx_error", "argmax_grid",
    "FactorPair", "Trajectory", "UpdateOutcome", "Orientation", "RunConfig", "random_acol_init",
    "f_ulf", "f_urf", "run_fit", "stmf_baseline", "StrategySpec", "BASELINE", "FASTSTMF",
    "parse_method", "fit", "fast_stmf", "FitSession", "build", "StmfError", "datagen", "io", "metrics", "__version__",
    "argmax_k", "b_norm", "sort_perm_by_min", "td", "td_col", "td_grid", "td_row", "SynthSpec", "apply_mask",
    "gen_mixture", "gen_tall_wide_pair", "NEVER", "bootstrap_ci", "distance_correlation", "masked_dc", "nemenyi_cd",
    "normalized_error", "omega", "rank_methods", "rmse", "time_to_reach",
]
