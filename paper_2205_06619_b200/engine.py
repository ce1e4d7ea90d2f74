"""Fitting engine: host orientation/initialisation + the device-resident sweep loop.

Mirrors the reference engine (engine.py) at its public names:
  * ``random_acol_init`` — RNG draws and column means on the host with numpy (the
    exact reference draw sequence, engine.py:170-195), the residuation
    V = (-U)^T (x)* R on the device;
  * ``run_fit`` — orient (host) -> init -> device sweeps -> restore (engine.py:313-348);
  * ``f_ulf`` / ``f_urf`` — single updates computed on the device, mutating U, V in
    place and returning an ``UpdateOutcome`` (engine.py:210-237).
Every method runs on the device kernels (FastSTMF as device-resident sweep graphs).
"""

from __future__ import annotations

import time

import numpy as np

from . import _ext
from .types import (FactorPair, MaskedMatrix, Orientation, Permutation, RunConfig, Trajectory,
                    UpdateOutcome)

__all__ = ["FitSession", "FitRun", "random_acol_init", "acol_means", "run_fit", "f_ulf", "f_urf",
           "stmf_baseline"]


class FitSession(_ext.Session):
    """Device state of one fit on a work-orientation ``MaskedMatrix``."""

    def __init__(self, work: MaskedMatrix, rank: int, device: int | None = None):
        super().__init__(work.values, work.mask, rank, device)


def acol_means(R: MaskedMatrix, rank: int, columns: int, rng: np.random.Generator) -> np.ndarray:
    """U of Random-Acol init: per factor column, the mean over given values of
    ``q = min(columns, n)`` data columns drawn with replacement, falling back to the
    row mean (engine.py:180-193).  Host numpy, same draws as the reference."""
    if rank < 1:
        raise ValueError("rank must be >= 1")
    q = min(columns, R.n)
    if q < 1:
        raise ValueError("need at least one column to average")
    row_fallback = R.row_means()
    vals64 = R.values.astype(np.float64, copy=False)
    U = np.empty((R.m, rank), dtype=np.float64)
    for c in range(rank):
        picks = rng.integers(0, R.n, size=q)
        given = R.mask[:, picks]
        vals = np.where(given, vals64[:, picks], 0.0)
        counts = given.sum(axis=1)
        with np.errstate(invalid="ignore", divide="ignore"):
            means = vals.sum(axis=1) / counts
        U[:, c] = np.where(counts > 0, means, row_fallback)
    return U.astype(R.dtype, copy=False)


def random_acol_init(R: MaskedMatrix, rank: int, columns: int, rng: np.random.Generator,
                     session: FitSession | None = None):
    """(U, V) of Random-Acol initialisation; V residuated on the device."""
    U = acol_means(R, rank, columns, rng)
    own = session is None
    s = FitSession(R, rank) if own else session
    try:
        s.set_factors(U)
        _, V = s.get_factors()
    finally:
        if own:
            s.close()
    return U, V


def _orient_faststmf(R: MaskedMatrix, rng: np.random.Generator):
    """_SpecStrategy.orient for ByRow/RandPermR/wide (strategies.py:324-337)."""
    transposed = R.m > R.n
    base = R.transpose() if transposed else R  # permute_rows returns fresh arrays: no copy first
    row_perm = Permutation.random(base.m, rng)
    work = base.permute_rows(row_perm)
    return work, Orientation(transposed, row_perm, None)


def _orient(spec, R: MaskedMatrix, rng: np.random.Generator):
    """strategy.orient: _SpecStrategy (strategies.py:324-337) or, for the STMF
    baseline, columns ascending by minimum without transposition (engine.py:361-363)."""
    from .strategies import BASELINE
    from .tropical import sort_perm_by_min
    if spec == BASELINE:
        perm = sort_perm_by_min(R, "cols")
        return R.permute_cols(perm), Orientation(col_perm=perm)
    transposed = spec.prefer_wide and R.m > R.n
    work = R.transpose() if transposed else R  # the permutations below return fresh arrays
    row_perm = col_perm = None
    if spec.permutation == "PermR":
        row_perm = sort_perm_by_min(work, "rows")
        work = work.permute_rows(row_perm)
    elif spec.permutation == "RandPermR":
        row_perm = Permutation.random(work.m, rng)
        work = work.permute_rows(row_perm)
    elif spec.permutation == "PermC":
        col_perm = sort_perm_by_min(work, "cols")
        work = work.permute_cols(col_perm)
    elif not transposed:
        work = R.copy()  # the fit never writes its input, but the caller's arrays stay the caller's
    return work, Orientation(transposed, row_perm, col_perm)


_SELECTION = {"TD_A": _ext.SEL_TD_A, "TD": _ext.SEL_TD, "TD_B": _ext.SEL_TD_B, "SEQ": _ext.SEL_SEQ}
_FAMILY = {"ByRow": _ext.FAMILY_BYROW, "ByElement": _ext.FAMILY_BYELEMENT, "ByMatrix": _ext.FAMILY_BYMATRIX}


def _strategy_codes(spec):
    from .strategies import BASELINE, StrategySpec
    if spec == BASELINE:
        return _ext.FAMILY_BASELINE, _ext.SEL_TD_A
    if not isinstance(spec, StrategySpec):
        raise NotImplementedError(f"unknown strategy {spec!r}")
    return _FAMILY[spec.family], _SELECTION[spec.selection] if spec.family == "ByRow" else _ext.SEL_TD_A


def _run_bymatrix(s: "FitSession", config: RunConfig, rng: np.random.Generator, t0: float):
    """run_fit's sweep loop (engine.py:328-344) with bymatrix_step (strategies.py:272-299)
    as the sweep.  The ranked candidate list and every attempt run on the device; the
    host only draws the reference's fair coin per candidate from the fit's RNG."""
    wall = config.budget_seconds is not None
    elapsed = (lambda: time.perf_counter() - t0) if wall else None
    sweep = 0

    def now():
        return elapsed() if wall else float(sweep)

    def out_of_time():
        return wall and elapsed() >= config.budget_seconds

    err = s.objective()
    tt, te = [now()], [err]
    attempts = accepts = sweeps = 0
    eps = config.epsilon * err
    if err > 0.0:
        while True:
            if config.budget_sweeps is not None and sweeps >= config.budget_sweeps:
                break
            if out_of_time():
                break
            sweep = sweeps + 1
            err_before = err
            rows, cols, ks, _ = s.matrix_candidates()
            for d in range(rows.size):
                if out_of_time():
                    break
                op = 0 if rng.random() < 0.5 else 1
                f, accepted = s.attempt(op, int(rows[d]), int(cols[d]), int(ks[d]))
                attempts += 1
                if accepted:
                    err = f
                    accepts += 1
                    tt.append(now())
                    te.append(err)
                    break
            sweeps += 1
            tt.append(now())
            te.append(err)
            if err_before - err < eps:
                break
    counts = {"traj_len": len(tt), "attempts": attempts, "accepts": accepts, "sweeps": sweeps,
              "row_visits": 0, "evaluated": 2 * attempts, "replicas": 0, "product_passes": 0}
    return np.array(tt), np.array(te), counts


def run_fit(R: MaskedMatrix, rank: int, strategy, config: RunConfig, device: int | None = None,
            init=None):
    """Budgeted outer loop (engine.py:313-348) with the sweeps on the device.

    ``strategy`` is a ``StrategySpec`` (or an object with ``.spec``) or ``BASELINE``
    ("STMF", the classic element-wise method, engine.py:351-385).  The FastSTMF
    strategy runs its sweeps as device-resident CUDA graphs; the other methods run
    the same device kernels under a host-driven batch loop.

    ``init`` (an extension; the reference always starts from Random-Acol): a warm
    start (U, V) or FactorPair in the original orientation, used instead of the Acol
    draws (the RNG stream then continues right after the orientation draws).
    """
    spec = getattr(strategy, "spec", strategy)
    family, selection = _strategy_codes(spec)
    if rank != config.rank:
        config = RunConfig(rank, config.budget_sweeps, config.budget_seconds, config.epsilon,
                           config.acol_columns, config.seed, config.audit)
    config.validate()
    R.validate_coverage()
    rng = np.random.default_rng(config.seed)
    wall_clock = config.budget_seconds is not None
    t0 = time.perf_counter()
    work, orientation = _orient(spec, R, rng)
    V0 = None
    if init is None:
        U0 = acol_means(work, rank, config.acol_columns, rng)
    else:
        Ui, Vi = (init.U, init.V) if isinstance(init, FactorPair) else init
        if np.shape(Ui) != (R.m, rank) or np.shape(Vi) != (rank, R.n):
            raise ValueError(f"init shapes {np.shape(Ui)}, {np.shape(Vi)} do not match {(R.m, rank)}, {(rank, R.n)}")
        U0, V0 = orientation.apply_factors(np.asarray(Ui, dtype=R.dtype), np.asarray(Vi, dtype=R.dtype))
    with FitSession(work, rank, device) as s:
        s.set_factors(U0, V0)
        if (family, selection) != (_ext.FAMILY_BYROW, _ext.SEL_TD_A):
            s.set_strategy(family, selection)
        if config.audit:
            # engine.py:279-294: the reference re-checks every revert; the device never
            # writes a rejected state, so it re-derives the committed one every sweep
            s.set_audit(True)
        t_init = time.perf_counter() - t0 if wall_clock else 0.0
        if family == _ext.FAMILY_BYMATRIX:
            tt, te, counts = _run_bymatrix(s, config, rng, time.perf_counter())
        else:
            budget_seconds = None
            if wall_clock:
                budget_seconds = max(config.budget_seconds - (time.perf_counter() - t0), 1e-9)
            # the trajectory is kept (growable) in the library and read back
            try:
                tt, te, counts = s.run(config.budget_sweeps, budget_seconds, config.epsilon)
            except _ext.StmfError as e:
                if e.code == 7:  # audit mismatch: the reference raises AssertionError (engine.py:294)
                    raise AssertionError(str(e)) from e
                raise
        U, V = s.get_factors()
    t_max = config.budget_seconds if wall_clock else float(config.budget_sweeps)
    traj = Trajectory(t_init=t_init, t_max=t_max, time_unit="seconds" if wall_clock else "sweeps")
    for t, e in zip(tt.tolist(), te.tolist()):
        traj.append(t + (t_init if wall_clock else 0.0), e)
    traj.counts = counts
    U_out, V_out = orientation.restore(U, V)
    return FactorPair(U_out, V_out, rank, orientation), traj


def _update(op: int, R: MaskedMatrix, U: np.ndarray, V: np.ndarray, i: int, j: int, k: int):
    if not R.mask[i, j]:
        raise ValueError(f"entry ({i}, {j}) is missing")
    saved_col = U[:, k].copy()
    saved_row = V[k, :].copy()
    with FitSession(R, U.shape[1]) as s:
        s.set_factors(U, V)
        ucol, vrow, f = s.try_update(op, i, j, k)
    U[:, k] = ucol
    V[k, :] = vrow
    return UpdateOutcome(f, k, saved_col, saved_row)


def f_ulf(R: MaskedMatrix, U: np.ndarray, V: np.ndarray, i: int, j: int, k: int) -> UpdateOutcome:
    """F-ULF at (i, j, k) on the device; mutates U, V (engine.py:210-225)."""
    return _update(0, R, U, V, i, j, k)


def f_urf(R: MaskedMatrix, U: np.ndarray, V: np.ndarray, i: int, j: int, k: int) -> UpdateOutcome:
    """F-URF at (i, j, k) on the device; mutates U, V (engine.py:228-237)."""
    return _update(1, R, U, V, i, j, k)


def stmf_baseline(R: MaskedMatrix, rank: int, config: RunConfig, device: int | None = None):
    """The original element-wise STMF (engine.py:383-385) on the device kernels."""
    from .strategies import BASELINE
    return run_fit(R, rank, BASELINE, config, device=device)


def __getattr__(name):  # engine.FitRun, as in the reference's engine module (engine.py:240-310)
    if name == "FitRun":
        from .fitrun import FitRun
        return FitRun
    raise AttributeError(name)
