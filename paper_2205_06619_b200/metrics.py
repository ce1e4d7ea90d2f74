"""The evaluation step after a fit (reference: metrics.py), on the device: prediction
error ``rmse`` (metrics.py:87-95) and ``distance_correlation`` / ``masked_dc``
(metrics.py:98-139).  Results are bit-identical to the reference's numpy (same
pairwise / sequential reduction trees; stmf_metrics.cuh).  The predictions come from
``FactorPair.product()`` (the device max-plus product, engine.py:86-87).

The trajectory statistics of metrics.py (normalized error on a time grid, bootstrap
intervals, method ranks, the Nemenyi critical difference, time-to-reach, the omega
shape statistic) post-process a handful of host floats: they are host numpy / scipy
here too, with the reference's semantics (metrics.py:33-206).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from . import _ext

__all__ = ["NEVER", "step_interpolate", "make_grid", "normalized_error", "rmse", "distance_correlation",
           "masked_dc", "bootstrap_ci", "rank_methods", "average_ranks", "nemenyi_cd", "time_to_reach", "omega",
           "NEGrid"]

#: "target never reached" (metrics.py:36); orders after every finite time
NEVER = math.inf


def rmse(pred, truth, mask) -> float:
    """Root-mean-square difference over the masked entries (0 if empty) (metrics.py:87-95)."""
    pred = np.asarray(pred, dtype=np.float64)
    truth = np.asarray(truth, dtype=np.float64)
    mask = np.asarray(mask, dtype=bool)
    if pred.ndim == 1:
        pred, truth, mask = pred[None, :], truth[None, :], mask[None, :]
    return _ext.masked_rmse(pred, truth, mask)


def distance_correlation(x, y) -> float:
    """Sample distance correlation of two equal-length 1-d samples (metrics.py:98-117)."""
    x = np.asarray(x, dtype=np.float64).ravel()
    y = np.asarray(y, dtype=np.float64).ravel()
    if x.size != y.size:
        raise ValueError("samples must have equal length")
    if x.size < 2:
        raise ValueError("need at least two samples")
    return _ext.distance_correlation(x, y)


def masked_dc(truth, approx, mask, max_entries: int = 2000, seed: int = 0) -> float:
    """Distance correlation between truth and approximation on a mask, subsampled
    (seeded, host RNG: the reference's draw) above ``max_entries`` (metrics.py:126-139)."""
    mask = np.asarray(mask, dtype=bool)
    x = np.asarray(truth, dtype=np.float64)[mask]
    y = np.asarray(approx, dtype=np.float64)[mask]
    if x.size > max_entries:
        idx = np.random.default_rng(seed).choice(x.size, size=max_entries, replace=False)
        x, y = x[idx], y[idx]
    return distance_correlation(x, y)


# ---- trajectory statistics (host) -------------------------------------------------

def step_interpolate(times, values, grid) -> np.ndarray:
    """Value of the last sample at or before each grid time; grid times before the
    first sample take the first value (metrics.py:39-49)."""
    t = np.asarray(times, dtype=np.float64)
    v = np.asarray(values, dtype=np.float64)
    if t.size == 0:
        raise ValueError("empty trajectory")
    pos = np.searchsorted(t, np.asarray(grid, dtype=np.float64), side="right") - 1
    return v[np.clip(pos, 0, None)]


def make_grid(t_max: float, step: float = 1.0, t_start: float = 0.0) -> np.ndarray:
    """t_start, t_start + step, ... up to t_max, with t_max itself appended when the
    steps fall short of it (metrics.py:52-60)."""
    if step <= 0:
        raise ValueError("step must be positive")
    count = int(math.floor((t_max - t_start) / step + 1e-9))
    grid = t_start + step * np.arange(count + 1)
    return grid if grid[-1] >= t_max else np.append(grid, t_max)


@dataclass
class NEGrid:
    """Normalized errors of several methods on one time grid (metrics.py:63-68)."""

    times: np.ndarray
    values: dict


def normalized_error(traj, baseline, grid) -> np.ndarray:
    """(error - baseline's error at its t_max) / (baseline's initial error - that), on the
    grid (metrics.py:69-84)."""
    final = step_interpolate(baseline.times, baseline.errors, [baseline.t_max])[0]
    span = baseline.init_error - final
    if span == 0.0:
        raise ValueError("degenerate baseline: error never changed")
    return (step_interpolate(traj.times, traj.errors, grid) - final) / span


def bootstrap_ci(samples, statistic=np.mean, n_resamples: int = 1000, level: float = 0.95,
                 seed: int = 0) -> tuple[float, float]:
    """Percentile interval of `statistic` over resamples with replacement
    (metrics.py:140-151; same draws: one integers() call of n_resamples x n)."""
    x = np.asarray(samples, dtype=np.float64)
    if x.size == 0:
        raise ValueError("no samples")
    draws = np.random.default_rng(seed).integers(0, x.size, size=(n_resamples, x.size))
    values = np.array([statistic(x[d]) for d in draws])
    tail = (1.0 - level) / 2.0
    lo, hi = np.quantile(values, [tail, 1.0 - tail])
    return float(lo), float(hi)


def rank_methods(scores, lower_is_better: bool = True) -> np.ndarray:
    """Ranks of a methods x datasets table per dataset column, ties averaged
    (metrics.py:154-166)."""
    from scipy.stats import rankdata
    table = np.asarray(scores, dtype=np.float64)
    if table.ndim != 2:
        raise ValueError("expected a methods x datasets table")
    keyed = table if lower_is_better else -table
    return np.stack([rankdata(keyed[:, j], method="average") for j in range(table.shape[1])], axis=1)


def average_ranks(rank_table) -> np.ndarray:
    """Mean rank of each method over the datasets (metrics.py:169-170)."""
    return np.asarray(rank_table, dtype=np.float64).mean(axis=1)


def nemenyi_cd(k: int, n_datasets: int, alpha: float = 0.05) -> float:
    """q_alpha * sqrt(k (k + 1) / (6 N)), q_alpha the infinite-dof studentized-range
    quantile over sqrt(2) (metrics.py:173-184)."""
    from scipy.stats import studentized_range
    if k < 2 or n_datasets < 1:
        raise ValueError("need k >= 2 methods and N >= 1 datasets")
    q = studentized_range.ppf(1.0 - alpha, k, np.inf) / math.sqrt(2.0)
    return float(q * math.sqrt(k * (k + 1) / (6.0 * n_datasets)))


def time_to_reach(traj, target: float, grid) -> float:
    """First grid time whose interpolated error is <= target, else NEVER
    (metrics.py:187-193)."""
    hit = np.flatnonzero(step_interpolate(traj.times, traj.errors, grid) <= target)
    return NEVER if hit.size == 0 else float(np.asarray(grid, dtype=np.float64)[hit[0]])


def omega(wide_errors, tall_errors) -> float:
    """Share of paired runs in which the wide orientation ended lower (metrics.py:196-206)."""
    w = np.asarray(wide_errors, dtype=np.float64)
    t = np.asarray(tall_errors, dtype=np.float64)
    if w.shape != t.shape or w.size == 0:
        raise ValueError("need equal-length nonempty error vectors")
    return float(np.mean(w < t))
