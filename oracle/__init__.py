"""TEST INFRASTRUCTURE ONLY — ctypes wrapper of the CPU restatement (oracle/*.c).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU-baseline legs may
import this package, and only as the checker / the reported CPU baseline.  The
product package (paper_2205_06619_b200) never imports it.

Every function mirrors a reference function (file:line in the C sources) on the
*work-orientation* arrays: X (m, n) with NaN under the mask, mask (m, n) bool,
U (m, r), V (r, n).  dtype float64 selects the numpy-compatible semantics,
float32 the exact-sum binary32 semantics (see stmf_oracle.h).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "libstmf_oracle.so")
_lib = None

_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double
_vp = ctypes.c_void_p


def build(force: bool = False) -> str:
    """Compile the restatement with its Makefile (gcc only; no reference sources)."""
    srcs = [os.path.join(_HERE, f) for f in ("stmf_oracle.c", "stmf_oracle_core.h", "stmf_oracle.h")]
    if force or not os.path.exists(_LIB_PATH) or any(
        os.path.getmtime(s) > os.path.getmtime(_LIB_PATH) for s in srcs
    ):
        subprocess.run(["make", "-C", _HERE, "-s"], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        L.orc_np_pairwise_sum.argtypes = [_vp, _i64]
        L.orc_np_pairwise_sum.restype = _dbl
        L.orc_b_norm_f64.argtypes = [_vp, _i64]
        L.orc_b_norm_f64.restype = _dbl
        L.orc_b_norm_f32.argtypes = [_vp, _i64]
        L.orc_b_norm_f32.restype = _dbl
        for s in ("f64", "f32"):
            getattr(L, f"orc_trop_matmul_{s}").argtypes = [_i64, _int, _i64, _vp, _vp, _vp, _vp, _vp]
            getattr(L, f"orc_residuate_row_{s}").argtypes = [_i64, _i64, _vp, _vp, _vp, _vp]
            getattr(L, f"orc_residuate_col_{s}").argtypes = [_i64, _i64, _vp, _vp, _vp, _vp]
            f = getattr(L, f"orc_approx_error_{s}")
            f.argtypes = [_i64, _int, _i64, _vp, _vp, _vp, _vp]
            f.restype = _dbl
            getattr(L, f"orc_col_scores_{s}").argtypes = [_i64, _int, _i64, _vp, _vp, _vp, _vp, _vp]
            for op in ("ulf", "urf"):
                f = getattr(L, f"orc_f_{op}_{s}")
                f.argtypes = [_i64, _int, _i64, _vp, _vp, _vp, _vp, _i64, _i64, _int, _vp]
                f.restype = _int
            f = getattr(L, f"orc_fit_{s}")
            f.argtypes = [_i64, _int, _i64, _vp, _vp, _vp, _vp, _i64, _dbl, _dbl, _i64,
                          _vp, _vp, _i64, _vp]
            f.restype = _int
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def _sfx(dtype) -> str:
    dtype = np.dtype(dtype)
    if dtype == np.float64:
        return "f64"
    if dtype == np.float32:
        return "f32"
    raise TypeError(f"unsupported dtype {dtype}")


def _prep(X, mask, dtype=None):
    X = np.asarray(X)
    dtype = np.dtype(dtype or X.dtype)
    X = np.ascontiguousarray(X, dtype=dtype)
    mask = np.ascontiguousarray(mask, dtype=np.uint8)
    return X, mask


def pairwise_sum(a) -> float:
    a = np.ascontiguousarray(a, dtype=np.float64)
    return lib().orc_np_pairwise_sum(_p(a), a.size)


def b_norm(vals) -> float:
    vals = np.asarray(vals)
    if vals.dtype == np.float32:
        v = np.ascontiguousarray(vals.ravel())
        return lib().orc_b_norm_f32(_p(v), v.size)
    v = np.ascontiguousarray(vals.ravel(), dtype=np.float64)
    return lib().orc_b_norm_f64(_p(v), v.size)


def trop_matmul(U, V):
    U = np.ascontiguousarray(U)
    V = np.ascontiguousarray(V, dtype=U.dtype)
    m, r = U.shape
    n = V.shape[1]
    P = np.empty((m, n), U.dtype)
    arg = np.empty((m, n), np.int32)
    top2 = np.empty((m, n), U.dtype)
    getattr(lib(), f"orc_trop_matmul_{_sfx(U.dtype)}")(m, r, n, _p(U), _p(V), _p(P), _p(arg), _p(top2))
    return P, arg, top2


def residuate_row(X, mask, u):
    X, mask = _prep(X, mask)
    u = np.ascontiguousarray(u, dtype=X.dtype)
    v = np.empty(X.shape[1], X.dtype)
    getattr(lib(), f"orc_residuate_row_{_sfx(X.dtype)}")(X.shape[0], X.shape[1], _p(X), _p(mask), _p(u), _p(v))
    return v


def residuate_col(X, mask, v):
    X, mask = _prep(X, mask)
    v = np.ascontiguousarray(v, dtype=X.dtype)
    u = np.empty(X.shape[0], X.dtype)
    getattr(lib(), f"orc_residuate_col_{_sfx(X.dtype)}")(X.shape[0], X.shape[1], _p(X), _p(mask), _p(v), _p(u))
    return u


def approx_error(X, mask, U, V) -> float:
    X, mask = _prep(X, mask)
    U = np.ascontiguousarray(U, dtype=X.dtype)
    V = np.ascontiguousarray(V, dtype=X.dtype)
    return getattr(lib(), f"orc_approx_error_{_sfx(X.dtype)}")(
        X.shape[0], U.shape[1], X.shape[1], _p(X), _p(mask), _p(U), _p(V))


def col_scores(X, mask, U, V):
    X, mask = _prep(X, mask)
    U = np.ascontiguousarray(U, dtype=X.dtype)
    V = np.ascontiguousarray(V, dtype=X.dtype)
    s = np.empty(X.shape[1], np.float64)
    getattr(lib(), f"orc_col_scores_{_sfx(X.dtype)}")(
        X.shape[0], U.shape[1], X.shape[1], _p(X), _p(mask), _p(U), _p(V), _p(s))
    return s


def _update(op, X, mask, U, V, i, j, k):
    X, mask = _prep(X, mask)
    U = np.array(U, dtype=X.dtype, order="C", copy=True)
    V = np.array(V, dtype=X.dtype, order="C", copy=True)
    f = ctypes.c_double()
    rc = getattr(lib(), f"orc_f_{op}_{_sfx(X.dtype)}")(
        X.shape[0], U.shape[1], X.shape[1], _p(X), _p(mask), _p(U), _p(V), i, j, k,
        ctypes.byref(f))
    if rc != 0:
        raise ValueError(f"entry ({i}, {j}) is missing")
    return U, V, f.value


def f_ulf(X, mask, U, V, i, j, k):
    """Returns (U', V', f) — engine.f_ulf (engine.py:210-225) on copies."""
    return _update("ulf", X, mask, U, V, i, j, k)


def f_urf(X, mask, U, V, i, j, k):
    """Returns (U', V', f) — engine.f_urf (engine.py:228-237) on copies."""
    return _update("urf", X, mask, U, V, i, j, k)


def fit(X, mask, U0, V0, budget_sweeps=None, budget_seconds=None, epsilon=1e-8,
        max_attempts=0, traj_cap=None):
    """run_fit after orientation + init (engine.py:327-344) with ByRow/TD_A sweeps."""
    X, mask = _prep(X, mask)
    U = np.array(U0, dtype=X.dtype, order="C", copy=True)
    V = np.array(V0, dtype=X.dtype, order="C", copy=True)
    m, n = X.shape
    if traj_cap is None:
        sweeps = budget_sweeps if budget_sweeps is not None else 1000
        traj_cap = 2 + (m + 1) * (sweeps + 1)
    tt = np.empty(traj_cap, np.float64)
    te = np.empty(traj_cap, np.float64)
    cnt = np.zeros(6, np.int64)
    rc = getattr(lib(), f"orc_fit_{_sfx(X.dtype)}")(
        m, U.shape[1], n, _p(X), _p(mask), _p(U), _p(V),
        -1 if budget_sweeps is None else int(budget_sweeps),
        0.0 if budget_seconds is None else float(budget_seconds),
        float(epsilon), int(max_attempts), _p(tt), _p(te), traj_cap, _p(cnt))
    if rc != 0:
        raise RuntimeError("trajectory capacity exceeded")
    L = int(cnt[0])
    return {
        "U": U, "V": V, "traj_t": tt[:L].copy(), "traj_err": te[:L].copy(),
        "attempts": int(cnt[1]), "accepts": int(cnt[2]), "sweeps": int(cnt[3]),
        "capped": bool(cnt[4]), "row_visits": int(cnt[5]),
    }
