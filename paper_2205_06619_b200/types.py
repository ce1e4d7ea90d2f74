"""Host-side data types of the drop-in API (same names, fields and errors as the
reference's tropical.py / engine.py types).

These hold host arrays only; all fitting arithmetic runs in the CUDA library.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

__all__ = ["Permutation", "MaskedMatrix", "Orientation", "FactorPair", "Trajectory",
           "UpdateOutcome", "RunConfig"]


@dataclass
class Permutation:
    """Permutation of 0..n-1 with its inverse (reference: tropical.py:32-63)."""

    forward: np.ndarray

    def __post_init__(self):
        fwd = np.asarray(self.forward, dtype=np.intp)
        if fwd.ndim != 1 or fwd.size == 0:
            raise ValueError("permutation must be a nonempty 1-d index array")
        n = fwd.size
        if fwd.min() < 0 or fwd.max() >= n:
            raise ValueError("permutation indices out of range")
        if np.unique(fwd).size != n:
            raise ValueError("permutation indices must be distinct")
        self.forward = fwd
        self.inverse = np.empty(n, dtype=np.intp)
        self.inverse[fwd] = np.arange(n, dtype=np.intp)

    @property
    def size(self) -> int:
        return self.forward.size

    @classmethod
    def identity(cls, n: int) -> "Permutation":
        return cls(np.arange(n, dtype=np.intp))

    @classmethod
    def random(cls, n: int, rng: np.random.Generator) -> "Permutation":
        # one rng.permutation(n) draw, as the reference (tropical.py:61-63)
        return cls(rng.permutation(n))


class MaskedMatrix:
    """Dense matrix with a boolean given-mask; NaN under the mask
    (reference: tropical.py:66-155).

    ``dtype`` (extension): float64 (default, the reference's storage and the
    numpy-compatible fit) or float32 (binary32 fit with exact-sum objective).
    """

    def __init__(self, values, mask=None, dtype=np.float64):
        dtype = np.dtype(dtype)
        if dtype not in (np.dtype(np.float64), np.dtype(np.float32)):
            raise ValueError("dtype must be float64 or float32")
        values = np.array(values, dtype=dtype)
        if values.ndim != 2:
            raise ValueError("expected a 2-d value array")
        if mask is None:
            mask = np.isfinite(values)
        mask = np.array(mask, dtype=bool)
        if mask.shape != values.shape:
            raise ValueError(f"mask shape {mask.shape} != value shape {values.shape}")
        if not np.isfinite(values[mask]).all():
            raise ValueError("given entries must be finite")
        values[~mask] = np.nan
        self.values = values
        self.mask = mask

    @property
    def dtype(self):
        return self.values.dtype

    @property
    def m(self) -> int:
        return self.values.shape[0]

    @property
    def n(self) -> int:
        return self.values.shape[1]

    @property
    def shape(self):
        return self.values.shape

    @property
    def given_count(self) -> int:
        return int(self.mask.sum())

    @classmethod
    def from_full(cls, values, dtype=np.float64) -> "MaskedMatrix":
        values = np.asarray(values, dtype=dtype)
        return cls(values, np.ones(values.shape, dtype=bool), dtype=dtype)

    @classmethod
    def _derived(cls, values: np.ndarray, mask: np.ndarray) -> "MaskedMatrix":
        """A matrix built from fresh copies of an already validated one (copy, transpose,
        permutation): the invariants (finite given entries, NaN under the mask) carry over,
        so the constructor's second copy and its passes over the data are skipped -- at
        config 3 they were 1.1 s of host time per fit (profiles/r02_e2e_host.md)."""
        obj = cls.__new__(cls)
        obj.values = values
        obj.mask = mask
        return obj

    def copy(self) -> "MaskedMatrix":
        return self._derived(self.values.copy(), self.mask.copy())

    def validate_coverage(self):
        if self.mask.size == 0:
            raise ValueError("empty matrix")
        rows = self.mask.any(axis=1)
        if not rows.all():
            raise ValueError(f"row {int(np.flatnonzero(~rows)[0])} has no given entries")
        cols = self.mask.any(axis=0)
        if not cols.all():
            raise ValueError(f"column {int(np.flatnonzero(~cols)[0])} has no given entries")

    def transpose(self) -> "MaskedMatrix":
        return self._derived(self.values.T.copy(), self.mask.T.copy())

    def permute_rows(self, p: Permutation) -> "MaskedMatrix":
        if p.size != self.m:
            raise ValueError("permutation length does not match row count")
        return self._derived(self.values[p.forward], self.mask[p.forward])

    def permute_cols(self, p: Permutation) -> "MaskedMatrix":
        if p.size != self.n:
            raise ValueError("permutation length does not match column count")
        return self._derived(self.values[:, p.forward], self.mask[:, p.forward])

    def row_mins(self) -> np.ndarray:
        """Per-row minimum over given entries, +inf for all-missing rows (tropical.py:141-143)."""
        return np.min(np.where(self.mask, self.values, np.inf), axis=1)

    def col_mins(self) -> np.ndarray:
        """Per-column minimum over given entries (tropical.py:145-146)."""
        return np.min(np.where(self.mask, self.values, np.inf), axis=0)

    def row_means(self) -> np.ndarray:
        """Per-row mean over given entries in float64 (reference: tropical.py:149-155)."""
        counts = self.mask.sum(axis=1)
        if (counts == 0).any():
            raise ValueError("row mean undefined for an all-missing row")
        sums = np.where(self.mask, self.values.astype(np.float64, copy=False), 0.0).sum(axis=1)
        return sums / counts


@dataclass
class Orientation:
    """Transforms applied before fitting (reference: engine.py:43-74)."""

    transposed: bool = False
    row_perm: Permutation | None = None
    col_perm: Permutation | None = None

    def apply(self, R: MaskedMatrix) -> MaskedMatrix:
        work = R.transpose() if self.transposed else R.copy()
        if self.row_perm is not None:
            work = work.permute_rows(self.row_perm)
        if self.col_perm is not None:
            work = work.permute_cols(self.col_perm)
        return work

    def apply_factors(self, U: np.ndarray, V: np.ndarray):
        """Factors of the original orientation -> the work orientation (inverse of
        ``restore``): a warm start's (U, V) for the work matrix ``apply(R)``."""
        U, V = np.asarray(U), np.asarray(V)
        if self.transposed:
            U, V = V.T, U.T
        if self.row_perm is not None:
            U = U[self.row_perm.forward, :]
        if self.col_perm is not None:
            V = V[:, self.col_perm.forward]
        return np.ascontiguousarray(U), np.ascontiguousarray(V)

    def restore(self, U: np.ndarray, V: np.ndarray):
        if self.row_perm is not None:
            U = U[self.row_perm.inverse, :]
        if self.col_perm is not None:
            V = V[:, self.col_perm.inverse]
        if self.transposed:
            U, V = V.T.copy(), U.T.copy()
        return np.ascontiguousarray(U), np.ascontiguousarray(V)

    def to_dict(self) -> dict:
        return {
            "transposed": self.transposed,
            "row_perm": None if self.row_perm is None else self.row_perm.forward.tolist(),
            "col_perm": None if self.col_perm is None else self.col_perm.forward.tolist(),
        }


@dataclass
class FactorPair:
    """U (m x r) and V (r x n) in the original orientation (reference: engine.py:77-87)."""

    U: np.ndarray
    V: np.ndarray
    rank: int
    orientation: Orientation = field(default_factory=Orientation)

    def product(self) -> np.ndarray:
        from .tropical import trop_matmul
        return trop_matmul(self.U, self.V)


class Trajectory:
    """Time-stamped non-increasing error samples (reference: engine.py:90-119)."""

    def __init__(self, t_init: float, t_max: float, time_unit: str = "seconds"):
        self.times: list[float] = []
        self.errors: list[float] = []
        self.t_init = t_init
        self.t_max = t_max
        self.time_unit = time_unit

    def append(self, t: float, err: float):
        if self.times and t < self.times[-1]:
            raise ValueError("timestamps must be non-decreasing")
        self.times.append(float(t))
        self.errors.append(float(err))

    @property
    def init_error(self) -> float:
        return self.errors[0]

    @property
    def final_error(self) -> float:
        return self.errors[-1]

    def __len__(self) -> int:
        return len(self.times)


@dataclass
class UpdateOutcome:
    """New error plus the saved column/row needed to undo the update (engine.py:122-133)."""

    f: float
    k: int
    saved_col: np.ndarray
    saved_row: np.ndarray

    def revert(self, U: np.ndarray, V: np.ndarray):
        U[:, self.k] = self.saved_col
        V[self.k, :] = self.saved_row


@dataclass
class RunConfig:
    """Knobs of one fitting run (reference: engine.py:136-167)."""

    rank: int
    budget_sweeps: int | None = None
    budget_seconds: float | None = None
    epsilon: float = 1e-8
    acol_columns: int = 5
    seed: int | None = None
    audit: bool = False

    def validate(self):
        if self.rank < 1:
            raise ValueError("rank must be >= 1")
        if self.budget_sweeps is None and self.budget_seconds is None:
            raise ValueError("set budget_sweeps or budget_seconds")
        if self.budget_sweeps is not None and self.budget_sweeps < 0:
            raise ValueError("budget_sweeps must be >= 0")
        if self.budget_seconds is not None and self.budget_seconds <= 0:
            raise ValueError("budget_seconds must be > 0")
        if self.acol_columns < 1:
            raise ValueError("acol_columns must be >= 1")
        if self.epsilon < 0:
            raise ValueError("epsilon must be >= 0")
