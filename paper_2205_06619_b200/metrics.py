"""The evaluation step after a fit (reference: metrics.py), on the device: prediction
error ``rmse`` (metrics.py:87-95) and ``distance_correlation`` / ``masked_dc``
(metrics.py:98-139).  Results are bit-identical to the reference's numpy (same
pairwise / sequential reduction trees; stmf_metrics.cuh).  The predictions come from
``FactorPair.product()`` (the device max-plus product, engine.py:86-87).

The trajectory statistics of metrics.py (normalized error, bootstrap intervals,
ranks, critical differences) post-process a handful of host floats and stay out of
scope.
"""

from __future__ import annotations

import numpy as np

from . import _ext

__all__ = ["rmse", "distance_correlation", "masked_dc"]


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
