"""Device versions of the reference's masked-matrix kernels used on the fit path
(tropical.py): the max-plus product with argmax, the masked min-plus residuation,
and the b-norm objective.  Host types live in ``types``.
"""

from __future__ import annotations

import numpy as np

from . import _ext
from .types import MaskedMatrix, Permutation

__all__ = ["MaskedMatrix", "Permutation", "trop_matmul", "argmax_grid", "approx_error",
           "masked_minplus", "sort_perm_by_min"]


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
