"""Device versions of the reference's masked-matrix kernels used on the fit path
(tropical.py): the max-plus product with argmax, the masked min-plus residuation,
and the b-norm objective.  Host types live in ``types``.
"""

from __future__ import annotations

import numpy as np

from . import _ext
from .types import MaskedMatrix, Permutation

__all__ = ["MaskedMatrix", "Permutation", "trop_matmul", "argmax_grid", "approx_error",
           "masked_minplus", "sort_perm_by_min", "b_norm", "td", "argmax_k", "td_row", "td_col", "td_grid"]


def trop_matmul(A, B) -> np.ndarray:
    """out[i, j] = max_k A[i, k] + B[k, j] (tropical.py:158-169), on the device."""
    return _ext.trop_matmul(A, B)


def argmax_grid(U, V) -> np.ndarray:
    """Lowest k attaining max_k U[i, k] + V[k, j] (tropical.py:260-262), on the device."""
    return _ext.trop_matmul(U, V, want_arg=True)[1].astype(np.intp)


def approx_error(R: MaskedMatrix, U, V) -> float:
    """b_norm(R - U (x) V) over given entries (tropical.py:214-222), on the device."""
    U = np.asarray(U, dtype=R.dtype)
    V = np.asarray(V, dtype=R.dtype)
    if U.shape[0] != R.m or V.shape[1] != R.n or U.shape[1] != V.shape[0]:
        raise ValueError(f"factor shapes {U.shape} x {V.shape} do not match data {R.shape}")
    with _ext.Session(R.values, R.mask, U.shape[1]) as s:
        s.set_factors(U, V)
        return s.objective()


def masked_minplus(negU_T, R: MaskedMatrix) -> np.ndarray:
    """(-U)^T (x)* R for a fully given U (the only use on the fit path,
    engine.py:194 -> tropical.py:179-194), on the device."""
    A = np.asarray(negU_T)
    U = -A.T
    out = np.empty((A.shape[0], R.n), R.dtype)
    with _ext.Session(R.values, R.mask, A.shape[0]) as s:
        for k in range(A.shape[0]):
            out[k] = s.residuate(0, U[:, k])
    return out


def sort_perm_by_min(M: MaskedMatrix, axis: str) -> Permutation:
    """Rows or columns ascending by their minimum over given entries, stable
    (tropical.py:265-277).  Host-side: part of the strategy's orientation, which
    runs once per fit before any device work."""
    if axis == "rows":
        mins = M.row_mins()
    elif axis == "cols":
        mins = M.col_mins()
    else:
        raise ValueError(f"axis must be 'rows' or 'cols', got {axis!r}")
    return Permutation(np.argsort(mins, kind="stable"))


def b_norm(W, mask=None) -> float:
    """Sum of |values| over the given entries, numpy's sorted pairwise sum, on the
    device (tropical.py:197-211); 0 for an empty mask."""
    if isinstance(W, MaskedMatrix):
        values, mask = W.values, W.mask
    else:
        values = np.asarray(W, dtype=np.float64)
    vals = np.asarray(values if mask is None else values[np.asarray(mask, dtype=bool)], dtype=np.float64)
    return 0.0 if vals.size == 0 else _ext.b_norm(vals)


def td_grid(R: MaskedMatrix, U, V, product=None) -> np.ndarray:
    """|R - U (x) V| at the given entries, 0 elsewhere (tropical.py:237-245); the product
    on the device unless given."""
    P = trop_matmul(U, V) if product is None else np.asarray(product)
    return np.where(R.mask, np.abs(np.where(R.mask, R.values, 0.0) - P), 0.0)


# Single-entry / single-line helpers of the reference (tropical.py:225-257): O(r) or
# O(n r) host arithmetic on a handful of values (used by the reference's non-FastSTMF
# strategies when driven by hand; the device engine computes the same quantities inside
# its kernels).
def td(R: MaskedMatrix, U, V, i: int, j: int) -> float:
    """|R[i, j] - max_k(U[i, k] + V[k, j])| of a given entry (tropical.py:225-229)."""
    if not R.mask[i, j]:
        raise ValueError(f"entry ({i}, {j}) is missing")
    return float(abs(R.values[i, j] - np.max(np.asarray(U)[i, :] + np.asarray(V)[:, j])))


def argmax_k(U, V, i: int, j: int) -> int:
    """Lowest k attaining max_k U[i, k] + V[k, j] (tropical.py:232-234)."""
    return int(np.argmax(np.asarray(U)[i, :] + np.asarray(V)[:, j]))


def td_row(R: MaskedMatrix, U, V, i: int) -> float:
    """Sum of the entry errors over the given entries of row i (tropical.py:248-251)."""
    p = np.max(np.asarray(U)[i, :][None, :] + np.asarray(V).T, axis=1)
    return float(np.sum(np.abs(R.values[i] - p)[R.mask[i]]))


def td_col(R: MaskedMatrix, U, V, j: int) -> float:
    """Sum of the entry errors over the given entries of column j (tropical.py:254-257)."""
    p = np.max(np.asarray(U) + np.asarray(V)[:, j][None, :], axis=1)
    return float(np.sum(np.abs(R.values[:, j] - p)[R.mask[:, j]]))
