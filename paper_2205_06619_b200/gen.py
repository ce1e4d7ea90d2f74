"""Seeded synthetic inputs for the five BASELINE.json configs.

All data is synthetic (the paper's TCGA data is not available); draws follow the
recipes in SURVEY.md §8d so C1/C2 coincide with the reference's datagen
(apply_mask: exact-count uniform hiding with coverage redraw, datagen.py:52-78).
Generation is host numpy (input side, not the fit path).
"""

from __future__ import annotations

import numpy as np

from .types import MaskedMatrix

__all__ = ["maxplus_host", "apply_mask", "config1", "config2", "config3", "config4", "CONFIGS"]

_MAX_REDRAWS = 1000


def maxplus_host(A: np.ndarray, B: np.ndarray, block: int = 1024) -> np.ndarray:
    """max_k A[i,k] + B[k,j] in numpy, row-blocked (data generation only)."""
    m = A.shape[0]
    out = np.empty((m, B.shape[1]), dtype=np.result_type(A, B))
    for r0 in range(0, m, block):
        a = A[r0:r0 + block]
        acc = a[:, 0:1] + B[0:1, :]
        for k in range(1, A.shape[1]):
            np.maximum(acc, a[:, k:k + 1] + B[k:k + 1, :], out=acc)
        out[r0:r0 + block] = acc
    return out


def apply_mask(X: np.ndarray, fraction: float, seed=None, dtype=np.float64):
    """Hide exactly floor(fraction*m*n) entries uniformly; redraw until every row and
    column keeps a given entry.  Same draws as the reference's apply_mask."""
    X = np.asarray(X)
    m, n = X.shape
    count = int(np.floor(fraction * m * n))
    if m * n - count < max(m, n):
        raise ValueError(f"masking {count} of {m * n} entries cannot leave every row and column a given entry")
    rng = seed if isinstance(seed, np.random.Generator) else np.random.default_rng(seed)
    for _ in range(_MAX_REDRAWS):
        hidden = np.zeros(m * n, dtype=bool)
        hidden[rng.choice(m * n, size=count, replace=False)] = True
        hidden = hidden.reshape(m, n)
        given = ~hidden
        if given.any(axis=1).all() and given.any(axis=0).all():
            return MaskedMatrix(X, given, dtype=dtype), hidden
    raise ValueError("could not draw a mask keeping every row and column covered")


def config1(seed: int = 0, mask_seed: int = 1) -> MaskedMatrix:
    """C1: 200x100, U,V~U[0,1) rank 3, max-plus + N(0,0.01), 20% hidden, fp64."""
    rng = np.random.default_rng(seed)
    A = rng.random((200, 3))
    B = rng.random((3, 100))
    X = maxplus_host(A, B) + rng.normal(0, 0.01, (200, 100))
    return apply_mask(X, 0.2, seed=mask_seed)[0]


def config2(seed: int = 0, mask_seed: int = 1) -> MaskedMatrix:
    """C2: 500x1000 log2(1 + lognormal(0, 1)), 50% hidden, fp64."""
    rng = np.random.default_rng(seed)
    X = np.log2(1 + rng.lognormal(0, 1, (500, 1000)))
    return apply_mask(X, 0.5, seed=mask_seed)[0]


def config3(seed: int = 0, mask_seed: int = 1, m: int = 4096, n: int = 8192, rank: int = 10) -> MaskedMatrix:
    """C3: 4096x8192 rank-10 max-plus + N(0, 0.05), 70% hidden, fp32 (generated in
    fp64, cast once)."""
    rng = np.random.default_rng(seed)
    A = rng.random((m, rank))
    B = rng.random((rank, n))
    X = maxplus_host(A, B)
    X += rng.normal(0, 0.05, (m, n))
    return apply_mask(X, 0.7, seed=mask_seed, dtype=np.float32)[0]


def config4(seed: int = 0, m: int = 32768, n: int = 32768, rank: int = 20, blocks: int = 64) -> MaskedMatrix:
    """C4: 32768^2 rank-20 max-plus + Laplace(0, 0.05); per-row missing rate
    p_i ~ Beta(9, 1), entries hidden iid with p_i; rows/columns left empty get
    one forced given entry.  fp32.  Row blocks use spawned generators so the
    result does not depend on memory limits."""
    ss = np.random.SeedSequence(seed)
    top, *kids = ss.spawn(blocks + 1)
    g = np.random.default_rng(top)
    A = g.random((m, rank))
    B = g.random((rank, n))
    p = g.beta(9.0, 1.0, size=m)
    X = np.empty((m, n), np.float32)
    M = np.empty((m, n), bool)
    edges = np.linspace(0, m, blocks + 1).astype(int)
    for b in range(blocks):
        r0, r1 = edges[b], edges[b + 1]
        gb = np.random.default_rng(kids[b])
        Xb = maxplus_host(A[r0:r1], B)
        Xb += gb.laplace(0, 0.05, (r1 - r0, n))
        X[r0:r1] = Xb
        M[r0:r1] = gb.random((r1 - r0, n)) >= p[r0:r1, None]
    rows = np.flatnonzero(~M.any(axis=1))
    fix = np.random.default_rng(ss.spawn(1)[0])
    for i in rows:
        M[i, fix.integers(0, n)] = True
    cols = np.flatnonzero(~M.any(axis=0))
    for j in cols:
        M[fix.integers(0, m), j] = True
    return MaskedMatrix(X, M, dtype=np.float32)


CONFIGS = {
    1: dict(make=config1, rank=3, sweeps=100, dtype="f64"),
    2: dict(make=config2, rank=5, sweeps=300, dtype="f64"),
    3: dict(make=config3, rank=10, sweeps=200, dtype="f32"),
    4: dict(make=config4, rank=20, sweeps=50, dtype="f32"),
}
