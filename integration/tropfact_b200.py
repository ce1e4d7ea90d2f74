"""The binding a tropfact maintainer would add: the reference's
run_fit (engine.py:313-348) for FastSTMF with the sweep loop in libstmf_b200.so, over
ctypes and the C ABI of include/stmf_b200.h only.  Host-side it keeps the reference's
own code: validation, the RNG stream, _SpecStrategy.orient, random_acol_init's draws,
Trajectory / FactorPair / Orientation.restore.

    import tropfact, tropfact_b200
    pair, traj = tropfact_b200.fast_stmf(tropfact, R, rank, config)

``tropfact`` is the reference package module (unmodified); nothing here imports this
repository's Python package.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.environ.get("STMF_LIB", os.path.join(_HERE, "..", "paper_2205_06619_b200", "lib", "libstmf_b200.so"))
_L = None
vp, i64, dbl, cint = ctypes.c_void_p, ctypes.c_int64, ctypes.c_double, ctypes.c_int


def lib():
    global _L
    if _L is None:
        L = ctypes.CDLL(LIB)
        L.stmf_create.argtypes = [ctypes.POINTER(vp), cint, i64, i64, cint, vp, vp, cint]
        L.stmf_set_factors.argtypes = [vp, vp, vp]
        L.stmf_run.argtypes = [vp, i64, dbl, dbl, vp, vp, i64, vp]
        L.stmf_trajectory.argtypes = [vp, vp, vp, i64, ctypes.POINTER(i64)]
        L.stmf_get_factors.argtypes = [vp, vp, vp]
        L.stmf_destroy.argtypes = [vp]
        L.stmf_last_error.restype = ctypes.c_char_p
        for f in ("stmf_create", "stmf_set_factors", "stmf_run", "stmf_trajectory", "stmf_get_factors",
                  "stmf_destroy"):
            getattr(L, f).restype = cint
        _L = L
    return _L


def _ck(rc: int):
    if rc:
        raise RuntimeError(f"stmf_b200 error {rc}: {lib().stmf_last_error().decode()}")


def run_fit_b200(tropfact, R, rank: int, config, device: int = 0):
    """engine.run_fit(R, rank, _SpecStrategy(FASTSTMF), config) with the sweeps on a B200."""
    import importlib
    eng = importlib.import_module(tropfact.__name__ + ".engine")
    strat = importlib.import_module(tropfact.__name__ + ".strategies")
    FactorPair, Trajectory, random_acol_init = eng.FactorPair, eng.Trajectory, eng.random_acol_init
    FASTSTMF, _SpecStrategy = strat.FASTSTMF, strat._SpecStrategy
    config.validate()                                   # engine.py:320
    R.validate_coverage()                               # engine.py:321
    rng = np.random.default_rng(config.seed)            # engine.py:322
    wall = config.budget_seconds is not None
    work, orientation = _SpecStrategy(FASTSTMF).orient(R, rng)        # strategies.py:324-337
    U0, _ = random_acol_init(work, rank, config.acol_columns, rng)    # host draws; V again on device
    X = np.ascontiguousarray(np.where(work.mask, work.values, 0.0), dtype=np.float64)
    M = np.ascontiguousarray(work.mask, dtype=np.uint8)
    h = vp()
    _ck(lib().stmf_create(ctypes.byref(h), 0, work.m, work.n, rank, X.ctypes.data, M.ctypes.data, device))
    try:
        _ck(lib().stmf_set_factors(h, np.ascontiguousarray(U0, dtype=np.float64).ctypes.data, None))
        cnt = np.zeros(8, np.int64)
        _ck(lib().stmf_run(h, -1 if config.budget_sweeps is None else int(config.budget_sweeps),
                           float(config.budget_seconds or 0.0), float(config.epsilon), None, None, 0,
                           cnt.ctypes.data))
        n = i64()
        _ck(lib().stmf_trajectory(h, None, None, 0, ctypes.byref(n)))
        tt, te = np.empty(n.value), np.empty(n.value)
        _ck(lib().stmf_trajectory(h, tt.ctypes.data, te.ctypes.data, n.value, ctypes.byref(n)))
        U = np.empty((work.m, rank))
        V = np.empty((rank, work.n))
        _ck(lib().stmf_get_factors(h, U.ctypes.data, V.ctypes.data))
    finally:
        lib().stmf_destroy(h)
    t_max = config.budget_seconds if wall else float(config.budget_sweeps)
    traj = Trajectory(0.0, t_max, "seconds" if wall else "sweeps")   # engine.py:259-262
    for t, e in zip(tt.tolist(), te.tolist()):
        traj.append(t, e)
    U, V = orientation.restore(U, V)                    # engine.py:346
    return FactorPair(U, V, rank, orientation), traj


def fast_stmf(tropfact, R, rank: int, config, device: int = 0):
    """strategies.fast_stmf (strategies.py:360-362) routed to the B200 engine."""
    return run_fit_b200(tropfact, R, rank, config, device)
