"""The reference's hand-driven fitting protocol on the device: ``FitRun`` (engine.py:240-310)
and the per-row / per-sweep strategy functions that drive it (strategies.py:147-314).

``run_fit`` does not go through these (it runs whole sweeps inside the library, as CUDA
graphs); they exist so that code written against the reference's lower-level names —
``FitRun.try_ulf`` / ``try_urf`` / ``trial``, ``byrow_sweep``, ``byrow_seq``,
``byelement_sweep``, ``bymatrix_step``, ``bymatrix_candidates``, ``select_k_td*`` — keeps
working.  Every update, objective, score and product is computed by the CUDA library
through the C ABI (``stmf_attempt``, ``stmf_try_update``, ``stmf_col_scores``,
``stmf_row_scores``, ``stmf_product_given``, ``stmf_matrix_candidates``); the host only
orders candidates and counts votes, as the reference's Python does.
"""

from __future__ import annotations

import time
from dataclasses import dataclass

import numpy as np

from . import _ext
from .types import MaskedMatrix, RunConfig, Trajectory

__all__ = ["FitRun", "UpdateCandidate", "select_k_td", "select_k_td_a", "select_k_td_b", "byrow_sweep",
           "byrow_seq", "byelement_sweep", "bymatrix_step", "bymatrix_candidates"]

_ULF, _URF = 0, 1


def _opcode(op) -> int:
    """f_ulf / f_urf (the functions, as the reference passes them), their names, or 0 / 1."""
    name = getattr(op, "__name__", op)
    if name in ("f_ulf", "ulf", _ULF):
        return _ULF
    if name in ("f_urf", "urf", _URF):
        return _URF
    raise ValueError(f"unknown update rule {op!r}")


@dataclass(frozen=True)
class UpdateCandidate:
    """A position to try, with the score that ranked it (strategies.py:67-74)."""

    i: int
    j: int
    k: int
    err_score: float


class FitRun:
    """Mutable state of one fitting run in its work orientation (engine.py:240-310).

    The state lives in a device session; ``U`` and ``V`` are the caller's arrays, updated
    in place after every accepted update (the reference mutates them in place too).  A
    rejected update never touches the committed state, so there is nothing to revert.
    """

    def __init__(self, R: MaskedMatrix, U: np.ndarray, V: np.ndarray, config: RunConfig, wall_clock: bool,
                 device: int | None = None):
        self.R = R
        self.U = U
        self.V = V
        self.config = config
        self.wall_clock = wall_clock
        self._t0 = time.perf_counter()
        self.current_sweep = 0
        self._s = _ext.Session(R.values, R.mask, U.shape[1], device)
        self._s.set_factors(np.ascontiguousarray(U, dtype=R.dtype), np.ascontiguousarray(V, dtype=R.dtype))
        self.err = self._s.objective()
        t_max = config.budget_seconds if wall_clock else float(config.budget_sweeps)
        self.trajectory = Trajectory(t_init=self.elapsed(), t_max=t_max,
                                     time_unit="seconds" if wall_clock else "sweeps")
        self.trajectory.append(self._now(), self.err)
        self.accepted_updates = 0
        self.attempted_updates = 0
        self._rows, self._cols = np.nonzero(R.mask)  # the given entries in the library's (row-major) order

    # -- lifetime -----------------------------------------------------------------
    def close(self):
        self._s.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # -- clock (engine.py:267-276) ---------------------------------------------------
    def elapsed(self) -> float:
        return time.perf_counter() - self._t0 if self.wall_clock else 0.0

    def _now(self) -> float:
        return self.elapsed() if self.wall_clock else float(self.current_sweep)

    def out_of_time(self) -> bool:
        return self.wall_clock and self.elapsed() >= self.config.budget_seconds

    # -- attempts (engine.py:278-310) --------------------------------------------------
    def _attempt(self, op, i: int, j: int, k: int) -> bool:
        if not self.R.mask[i, j]:
            raise ValueError(f"entry ({i}, {j}) is missing")
        f, accepted = self._s.attempt(_opcode(op), int(i), int(j), int(k))
        self.attempted_updates += 1
        if accepted:
            self.err = f
            self.accepted_updates += 1
            self.trajectory.append(self._now(), self.err)
            U, V = self._s.get_factors()  # only column k of U and row k of V changed
            self.U[:, k] = U[:, k]
            self.V[k, :] = V[k, :]
        return accepted

    def try_ulf(self, i: int, j: int, k: int) -> bool:
        return self._attempt(_ULF, i, j, k)

    def try_urf(self, i: int, j: int, k: int) -> bool:
        return self._attempt(_URF, i, j, k)

    def trial(self, op, i: int, j: int, k: int) -> float:
        """The error an update would give; records and changes nothing (engine.py:303-307)."""
        if not self.R.mask[i, j]:
            raise ValueError(f"entry ({i}, {j}) is missing")
        return self._s.try_update(_opcode(op), int(i), int(j), int(k))[2]

    def mark_sweep_boundary(self):
        self.trajectory.append(self._now(), self.err)

    # -- device views used by the strategy functions ---------------------------------
    def _arg_grid(self) -> np.ndarray:
        """argmax_grid(U, V) at the given entries (-1 elsewhere), from the device caches."""
        _, arg, _ = self._s.product_given()
        g = np.full(self.R.shape, -1, dtype=np.intp)
        g[self._rows, self._cols] = arg
        return g


def _pair_max(U, V, i: int, j: int):
    return np.max(np.asarray(U)[i, :] + np.asarray(V)[:, j])


def select_k_td(U, V, i: int, j: int) -> int:
    """Factor index attaining max_k(U[i, k] + V[k, j]); smallest on ties (strategies.py:147-149)."""
    return int(np.argmax(np.asarray(U)[i, :] + np.asarray(V)[:, j]))


def _vote(votes: np.ndarray, rank: int) -> int:
    return int(np.argmax(np.bincount(votes, minlength=rank)))


def _session_for(R: MaskedMatrix, U, V) -> _ext.Session:
    s = _ext.Session(R.values, R.mask, np.shape(U)[1])
    s.set_factors(np.ascontiguousarray(U, dtype=R.dtype), np.ascontiguousarray(V, dtype=R.dtype))
    return s


def select_k_td_a(R: MaskedMatrix, U, V, i: int, j: int) -> int:
    """Most frequent argmax index among the given entries of row i and column j; smallest
    index on tied counts (strategies.py:152-157).  The argmax indices come from the device."""
    with _session_for(R, U, V) as s:
        _, arg, _ = s.product_given()
    rows, cols = np.nonzero(R.mask)
    votes = np.concatenate([arg[rows == i], arg[cols == j]])
    return _vote(votes, np.shape(U)[1])


def _select_td_b(U, V, row_scores, col_scores, i: int, j: int) -> int:
    j0 = int(np.argmax(col_scores))
    i0 = int(np.argmax(row_scores))
    if _pair_max(U, V, i, j0) >= _pair_max(U, V, i0, j):
        return select_k_td(U, V, i, j0)
    return select_k_td(U, V, i0, j)


def select_k_td_b(R: MaskedMatrix, U, V, i: int, j: int) -> int:
    """k at the row or column where the scan scores peak (strategies.py:164-177): j0 / i0
    maximise the column / row error totals (device), the index comes from whichever of
    (i, j0), (i0, j) has the larger approximation value, the row scan on ties."""
    with _session_for(R, U, V) as s:
        col_scores, row_scores = s.col_scores(), s.row_scores()
    return _select_td_b(U, V, row_scores, col_scores, i, j)


def _ranked_row_candidates(run: FitRun, i: int):
    """Given columns of row i by decreasing column score, stable (strategies.py:183-188)."""
    scores = run._s.col_scores()
    cols = np.flatnonzero(run.R.mask[i, :])
    order = np.argsort(-scores[cols], kind="stable")
    return cols[order], scores


def byrow_sweep(run: FitRun, i: int, selection: str) -> bool:
    """Try the candidates of row i in score order until one update sticks: F-ULF, then
    F-URF at the same position (strategies.py:191-224)."""
    if selection == "SEQ":
        return byrow_seq(run, i)
    if selection not in ("TD", "TD_A", "TD_B"):
        raise ValueError(f"unknown selection {selection!r}")
    R, U, V = run.R, run.U, run.V
    cols, col_scores = _ranked_row_candidates(run, i)
    if selection == "TD_A":
        arg = run._arg_grid()
        row_votes = arg[i, R.mask[i, :]]
        rank = U.shape[1]
    elif selection == "TD_B":
        row_scores = run._s.row_scores()
    for j in cols.tolist():
        if selection == "TD":
            k = select_k_td(U, V, i, j)
        elif selection == "TD_A":
            k = _vote(np.concatenate([row_votes, arg[R.mask[:, j], j]]), rank)
        else:
            k = _select_td_b(U, V, row_scores, col_scores, i, j)
        if run.try_ulf(i, j, k):
            return True
        if run.try_urf(i, j, k):
            return True
        if run.out_of_time():
            return False
    return False


def byrow_seq(run: FitRun, i: int) -> bool:
    """Exhaustive row update (strategies.py:227-249): trial every (j, k, rule), apply the
    largest strict decrease (ties: smallest j, then k, then F-ULF)."""
    best = None
    cols = np.flatnonzero(run.R.mask[i, :])
    for j in cols.tolist():
        for k in range(run.U.shape[1]):
            for op in (_ULF, _URF):
                f = run.trial(op, i, j, k)
                if f < run.err and (best is None or f < best[0]):
                    best = (f, j, k, op)
    if best is None:
        return False
    _, j, k, op = best
    if not run._attempt(op, i, j, k):
        raise AssertionError("re-applying a strictly improving trial failed")
    return True


def byelement_sweep(run: FitRun) -> None:
    """Every given entry once, row-major (strategies.py:252-269): skip exact entries, k =
    the local argmax, F-ULF then F-URF, at most one accepted update per entry."""
    R, U, V = run.R, run.U, run.V
    for i, j in zip(run._rows.tolist(), run._cols.tolist()):
        if run.out_of_time():
            return
        sums = U[i, :] + V[:, j]
        k = int(np.argmax(sums))
        if abs(R.values[i, j] - sums[k]) == 0.0:
            continue
        if not run.try_ulf(i, j, k):
            run.try_urf(i, j, k)


def bymatrix_candidates(run: FitRun) -> list[UpdateCandidate]:
    """Scored candidate list of a whole-matrix step, in trial order (strategies.py:301-314);
    scores, argmax indices and the stable ranking are computed on the device."""
    rows, cols, ks, scores = run._s.matrix_candidates()
    return [UpdateCandidate(int(i), int(j), int(k), float(sc))
            for i, j, k, sc in zip(rows.tolist(), cols.tolist(), ks.tolist(), scores.tolist())]


def bymatrix_step(run: FitRun, rng: np.random.Generator) -> bool:
    """One whole-matrix step (strategies.py:272-299): candidates by decreasing score, the
    rule by a fair coin per candidate, until one update is accepted."""
    rows, cols, ks, _ = run._s.matrix_candidates()
    for d in range(rows.size):
        if run.out_of_time():
            return False
        op = _ULF if rng.random() < 0.5 else _URF
        if run._attempt(op, int(rows[d]), int(cols[d]), int(ks[d])):
            return True
    return False
