"""ctypes binding of libstmf_b200.so (include/stmf_b200.h).

The product path has no CPU fallback: if the library is missing or no CUDA device
is usable, every entry point raises.  ``build()`` compiles the library in-tree for
sm_100a (nvcc cross-compiles without a GPU).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
REPO_DIR = os.path.dirname(PKG_DIR)
LIB_PATH = os.path.join(PKG_DIR, "lib", "libstmf_b200.so")
CSRC = os.path.join(PKG_DIR, "csrc")
INCLUDE = os.path.join(REPO_DIR, "include")
SOURCES = ["stmf_api.cu", "stmf_io.cc"]
HEADERS = ["stmf_kernels.cuh", "stmf_shard.cuh", "stmf_maxplus.cuh", "stmf_graph.cuh", "stmf_strategies.cuh",
           "stmf_metrics.cuh", "stmf_fast1.cuh", "stmf_maxplus_lanes.cuh"]

STMF_F64, STMF_F32 = 0, 1
ERR_NAMES = {1: "invalid argument", 2: "CUDA error", 3: "out of device memory", 4: "numeric",
             5: "capacity", 6: "NCCL error", 7: "audit"}

NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]


class StmfError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"stmf_b200 {ERR_NAMES.get(code, code)}: {msg}")
        self.code = code


def _nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def nccl_include() -> str:
    """nccl.h of the pip NCCL that torch loads (the library itself is dlopen'ed)."""
    try:
        import nvidia.nccl
        base = list(nvidia.nccl.__path__)[0]
        inc = os.path.join(base, "include")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc
    except ImportError:
        pass
    for c in ("/usr/include", "/usr/local/cuda/include"):
        if os.path.exists(os.path.join(c, "nccl.h")):
            return c
    raise RuntimeError("nccl.h not found")


CHECKED_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib", "libstmf_b200_checked.so")


def build(force: bool = False, verbose: bool = False, out: str | None = None, defines=(),
          checked: bool = False) -> str:
    """Compile csrc/*.cu into lib/libstmf_b200.so for sm_100a (in-tree).  ``out`` /
    ``defines``: an experiment variant of the library (loaded with STMF_LIB).
    ``checked``: lib/libstmf_b200_checked.so with device-side index range checks
    (STMF_CHECKS; load it with STMF_LIB)."""
    if checked:
        out = out or CHECKED_LIB_PATH
        defines = tuple(defines) + ("STMF_CHECKS",)
    out = out or LIB_PATH
    srcs = [os.path.join(CSRC, s) for s in SOURCES]
    deps = srcs + [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(INCLUDE, "stmf_b200.h")]
    if not force and os.path.exists(out) and all(
            os.path.getmtime(d) <= os.path.getmtime(out) for d in deps):
        return out
    os.makedirs(os.path.dirname(out), exist_ok=True)
    tmp = out + ".tmp"
    cmd = [_nvcc(), *NVCC_FLAGS, *(f"-D{d}" for d in defines), "-I", INCLUDE, "-I", CSRC, "-I",
           nccl_include(), "-o", tmp, *srcs]
    if verbose:
        print(" ".join(cmd))
    subprocess.run(cmd, check=True)
    os.replace(tmp, out)
    return out


_lib = None
_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_int = ctypes.c_int
_dbl = ctypes.c_double


def lib():
    global _lib
    if _lib is not None:
        return _lib
    # STMF_LIB: an alternative in-tree build of the same library (kernel variants
    # compiled with other -D settings, for A/B measurements)
    path = os.environ.get("STMF_LIB") or LIB_PATH
    if not os.path.exists(path):
        raise StmfError(2, f"CUDA extension not built ({path} missing); run "
                           "paper_2205_06619_b200._ext.build() — there is no CPU fallback")
    L = ctypes.CDLL(path)
    L.stmf_last_error.restype = ctypes.c_char_p
    L.stmf_version.restype = ctypes.c_char_p
    sig = {
        "stmf_create": [ctypes.POINTER(_vp), _int, _i64, _i64, _int, _vp, _vp, _int],
        "stmf_destroy": [_vp],
        "stmf_info": [_vp, _vp],
        "stmf_set_factors": [_vp, _vp, _vp],
        "stmf_get_factors": [_vp, _vp, _vp],
        "stmf_objective": [_vp, ctypes.POINTER(_dbl)],
        "stmf_run": [_vp, _i64, _dbl, _dbl, _vp, _vp, _i64, _vp],
        "stmf_product_given": [_vp, _vp, _vp, _vp],
        "stmf_col_scores": [_vp, _vp],
        "stmf_residuate": [_vp, _int, _vp, _vp],
        "stmf_try_update": [_vp, _int, _i64, _i64, _int, _vp, _vp, ctypes.POINTER(_dbl)],
        "stmf_attempt": [_vp, _int, _i64, _i64, _int, ctypes.POINTER(_dbl), ctypes.POINTER(_int)],
        "stmf_bench_product": [_vp, _int, _int, ctypes.POINTER(_dbl), ctypes.POINTER(_dbl)],
        "stmf_trop_matmul": [_int, _i64, _int, _i64, _vp, _vp, _vp, _vp, _int],
        "stmf_stream": [_vp, ctypes.POINTER(_vp)],
        "stmf_set_profiling": [_vp, _int],
        "stmf_counters": [_vp, _vp],
        "stmf_nccl_unique_id": [_vp, ctypes.POINTER(_i64)],
        "stmf_create_sharded": [ctypes.POINTER(_vp), _int, _i64, _i64, _int, _vp, _vp, _vp, _vp, _int, _int,
                                _vp, _int],
        "stmf_create_sim_group": [ctypes.POINTER(_vp), _int, _i64, _i64, _int, _vp, _vp, _int, _int],
        "stmf_bench_maxplus": [_i64, _i64, _int, _dbl, ctypes.c_uint64, _int, _int, _int, _vp, _vp, _vp, _vp,
                               _vp],
        "stmf_bench_maxplus_layout": [_i64, _i64, _int, _dbl, ctypes.c_uint64, _int, _int, _int, _int, _vp, _vp,
                                      _vp, _vp, _vp],
        "stmf_set_strategy": [_vp, _int, _int],
        "stmf_row_scores": [_vp, _vp],
        "stmf_matrix_candidates": [_vp, _vp, _vp, _vp, _vp],
        "stmf_masked_rmse": [_i64, _i64, _vp, _vp, _vp, _int, ctypes.POINTER(_dbl)],
        "stmf_distance_correlation": [_i64, _vp, _vp, _int, ctypes.POINTER(_dbl)],
        "stmf_csv_open": [ctypes.c_char_p, _int, ctypes.POINTER(_vp), ctypes.POINTER(_i64), ctypes.POINTER(_i64)],
        "stmf_csv_fill": [_vp, _vp, _vp, _int],
        "stmf_csv_close": [_vp],
        "stmf_release_memory": [_int],
        "stmf_trajectory": [_vp, _vp, _vp, _i64, ctypes.POINTER(_i64)],
        "stmf_replayed_sweeps": [_vp, ctypes.POINTER(_i64)],
        "stmf_set_max_attempts": [_vp, _i64],
        "stmf_set_audit": [_vp, _int],
        "stmf_comm_info": [_vp, _vp],
        "stmf_b_norm": [_i64, _vp, _int, ctypes.POINTER(_dbl)],
    }
    for name, args in sig.items():
        f = getattr(L, name)
        f.argtypes = args
        f.restype = _int
    _lib = L
    return L


EXPORTED_SYMBOLS = ["stmf_last_error", "stmf_version", "stmf_create", "stmf_destroy", "stmf_info",
                    "stmf_set_factors", "stmf_get_factors", "stmf_objective", "stmf_run",
                    "stmf_product_given", "stmf_col_scores", "stmf_residuate", "stmf_try_update",
                    "stmf_attempt", "stmf_bench_product", "stmf_trop_matmul",
                    "stmf_stream", "stmf_set_profiling", "stmf_counters", "stmf_nccl_unique_id",
                    "stmf_create_sharded", "stmf_create_sim_group", "stmf_bench_maxplus", "stmf_bench_maxplus_layout",
                    "stmf_set_strategy", "stmf_row_scores", "stmf_matrix_candidates",
                    "stmf_masked_rmse", "stmf_distance_correlation", "stmf_csv_open", "stmf_csv_fill",
                    "stmf_csv_close", "stmf_release_memory",
                    "stmf_trajectory", "stmf_replayed_sweeps", "stmf_set_max_attempts", "stmf_set_audit", "stmf_comm_info",
                    "stmf_b_norm"]

# include/stmf_b200.h: families and ByRow selection rules
FAMILY_BYROW, FAMILY_BYELEMENT, FAMILY_BASELINE, FAMILY_BYMATRIX = 0, 1, 2, 3
SEL_TD_A, SEL_TD, SEL_TD_B, SEL_SEQ = 0, 1, 2, 3


def bench_maxplus(m: int, n: int, rank: int, density: float, seed: int = 0, reps: int = 5,
                  flush_l2: bool = True, device: int | None = None, want_data: bool = False, layout: str = "dense"):
    """Config-5 masked max-plus product + error microbench on device-generated data.
    layout: "dense" (k_maxplus_err), "sampled" (given values only: the lane-compacted kernel
    k_maxplus_err_lanes when n % 1024 == 0 and rank <= 16, else the tile kernel
    k_maxplus_err_sampled), "lanes" / "tiles" (demand one of the two sampled kernels) or
    "auto" (sampled at density <= 0.35).  The result's "kernel" names the one that ran."""
    code = {"dense": 0, "sampled": 1, "auto": -1, "lanes": 2, "tiles": 1}[layout]
    prev = os.environ.get("STMF_C5_SAMPLED")
    if layout == "tiles":
        os.environ["STMF_C5_SAMPLED"] = "tiles"
    out = np.zeros(8, np.float64)
    X = np.empty((m, n), np.float32) if want_data else None
    M = np.empty(m * n // 32, np.uint32) if want_data else None
    U = np.empty((rank, m), np.float32) if want_data else None
    V = np.empty((rank, n), np.float32) if want_data else None
    p = lambda a: None if a is None else _p(a)  # noqa: E731
    try:
        _check(lib().stmf_bench_maxplus_layout(m, n, rank, float(density), int(seed), int(reps), int(flush_l2),
                                               default_device() if device is None else int(device), code, _p(out),
                                               p(X), p(M), p(U), p(V)))
    finally:
        if layout == "tiles":
            if prev is None:
                os.environ.pop("STMF_C5_SAMPLED", None)
            else:
                os.environ["STMF_C5_SAMPLED"] = prev
    res = dict(zip(("avg_ms", "best_ms", "objective", "given", "gbs", "gpairs_per_s", "layout", "bytes"),
                   out.tolist()))
    res["kernel"] = {0: "k_maxplus_err", 1: "k_maxplus_err_sampled", 2: "k_maxplus_err_lanes"}[int(res["layout"])]
    res["layout"] = "sampled" if res["layout"] >= 1 else "dense"
    if want_data:
        mask = np.unpackbits(M.view(np.uint8), bitorder="little").reshape(m, n).astype(bool)
        res["data"] = (X, mask, U.T.copy(), V)
    return res


def _check(rc: int):
    if rc != 0:
        raise StmfError(rc, lib().stmf_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(_vp)


def dtype_code(dtype) -> int:
    dtype = np.dtype(dtype)
    if dtype == np.float64:
        return STMF_F64
    if dtype == np.float32:
        return STMF_F32
    raise TypeError(f"unsupported dtype {dtype} (float64 or float32)")


def trop_matmul(U, V, device: int | None = None, want_arg: bool = False):
    """Dense max-plus product (and lowest argmax) of host arrays on the device."""
    U = np.asarray(U)
    dtype = np.float32 if U.dtype == np.float32 else np.float64
    U = np.ascontiguousarray(U, dtype=dtype)
    V = np.ascontiguousarray(V, dtype=dtype)
    if U.ndim != 2 or V.ndim != 2 or U.shape[1] != V.shape[0]:
        raise ValueError(f"inner dimensions differ: {U.shape} x {V.shape}")
    m, r = U.shape
    n = V.shape[1]
    P = np.empty((m, n), dtype)
    arg = np.empty((m, n), np.int32) if want_arg else None
    _check(lib().stmf_trop_matmul(dtype_code(dtype), m, r, n, _p(U), _p(V), _p(P),
                                  None if arg is None else _p(arg),
                                  default_device() if device is None else int(device)))
    return (P, arg) if want_arg else P


def default_device() -> int:
    for var in ("STMF_DEVICE", "LOCAL_RANK"):
        if os.environ.get(var):
            return int(os.environ[var])
    return 0


def _host_inputs(X, mask, dtype):
    """The arrays handed to stmf_create*: X as is (the library ignores values under the mask,
    include/stmf_b200.h, so NaNs there need no scrubbing pass) and the boolean mask viewed as
    bytes; copies only when the layout or dtype requires one."""
    Xc = np.ascontiguousarray(X, dtype=dtype)
    mask = np.asarray(mask)
    if mask.shape != Xc.shape:
        raise ValueError(f"mask shape {mask.shape} != value shape {Xc.shape}")
    if mask.dtype == np.bool_ and mask.flags.c_contiguous:
        Mc = mask.view(np.uint8)
    else:
        Mc = np.ascontiguousarray(mask != 0, dtype=np.uint8)
    return Xc, Mc


class Session:
    """One device-resident fit state (work orientation).  Owns all device buffers."""

    def __init__(self, X: np.ndarray, mask: np.ndarray, rank: int, device: int | None = None):
        X = np.asarray(X)
        self.dtype = np.dtype(X.dtype)
        code = dtype_code(self.dtype)
        Xc, Mc = _host_inputs(X, mask, self.dtype)
        self.m, self.n = Xc.shape
        self.rank = int(rank)
        h = _vp()
        _check(lib().stmf_create(ctypes.byref(h), code, self.m, self.n, self.rank, _p(Xc), _p(Mc),
                                 default_device() if device is None else int(device)))
        self.sharded = False
        self._adopt(h)

    def _adopt(self, h):
        self._h = h
        info = np.zeros(5, np.int64)
        _check(lib().stmf_info(self._h, _p(info)))
        self.m, self.n, self.rank, self.given = (int(x) for x in info[:4])
        self.local_rows = self.m

    @classmethod
    def sim_group(cls, X, mask, rank: int, shards: int, device: int | None = None) -> "Session":
        """Row-sharded engine with `shards` row blocks in this process (one device)."""
        self = cls.__new__(cls)
        self.dtype = np.dtype(np.float32)
        Xc, Mc = _host_inputs(X, mask, np.float32)
        h = _vp()
        _check(lib().stmf_create_sim_group(ctypes.byref(h), STMF_F32, Xc.shape[0], Xc.shape[1], int(rank),
                                           _p(Xc), _p(Mc), int(shards),
                                           default_device() if device is None else int(device)))
        self.sharded = True
        self._adopt(h)
        return self

    @classmethod
    def sharded(cls, X_rows, mask_rows, rank: int, m: int, row_starts, row_nnz, world: int, shard: int,
                nccl_id: bytes | None, device: int | None = None) -> "Session":
        """This process's shard of a row-sharded fit (one GPU per process, NCCL)."""
        self = cls.__new__(cls)
        self.dtype = np.dtype(np.float32)
        Xc, Mc = _host_inputs(X_rows, mask_rows, np.float32)
        starts = np.ascontiguousarray(row_starts, dtype=np.int64)
        nnz = np.ascontiguousarray(row_nnz, dtype=np.int64)
        idbuf = None if nccl_id is None else ctypes.create_string_buffer(bytes(nccl_id), len(nccl_id))
        h = _vp()
        _check(lib().stmf_create_sharded(ctypes.byref(h), STMF_F32, int(m), Xc.shape[1], int(rank), _p(starts),
                                         _p(nnz), _p(Xc), _p(Mc), int(world), int(shard),
                                         None if idbuf is None else ctypes.cast(idbuf, _vp),
                                         default_device() if device is None else int(device)))
        self.sharded = True
        self._adopt(h)
        self.local_rows = Xc.shape[0]
        return self

    def close(self):
        if getattr(self, "_h", None):
            lib().stmf_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # factors ---------------------------------------------------------------
    def set_factors(self, U, V=None):
        U = np.ascontiguousarray(U, dtype=self.dtype)
        if U.shape != (self.local_rows, self.rank):
            raise ValueError(f"U shape {U.shape} != {(self.local_rows, self.rank)}")
        if V is not None:
            V = np.ascontiguousarray(V, dtype=self.dtype)
            if V.shape != (self.rank, self.n):
                raise ValueError(f"V shape {V.shape} != {(self.rank, self.n)}")
        _check(lib().stmf_set_factors(self._h, _p(U), None if V is None else _p(V)))

    def get_factors(self):
        U = np.empty((self.local_rows, self.rank), self.dtype)
        V = np.empty((self.rank, self.n), self.dtype)
        _check(lib().stmf_get_factors(self._h, _p(U), _p(V)))
        return U, V

    def objective(self) -> float:
        e = _dbl()
        _check(lib().stmf_objective(self._h, ctypes.byref(e)))
        return e.value

    def run(self, budget_sweeps=None, budget_seconds=None, epsilon=1e-8, traj_cap=None):
        """run_fit's sweep loop on the device.  traj_cap=None: the trajectory is kept in
        the library (growable) and read back after the run (single-device sessions);
        otherwise it goes to buffers of traj_cap samples."""
        counts = np.zeros(8, np.int64)
        bs = -1 if budget_sweeps is None else int(budget_sweeps)
        secs = 0.0 if budget_seconds is None else float(budget_seconds)
        if traj_cap is None:
            _check(lib().stmf_run(self._h, bs, secs, float(epsilon), None, None, 0, _p(counts)))
            L = int(counts[0])
            tt = np.empty(L, np.float64)
            te = np.empty(L, np.float64)
            n = _i64()
            _check(lib().stmf_trajectory(self._h, _p(tt), _p(te), L, ctypes.byref(n)))
        else:
            if traj_cap is None:
                sw = budget_sweeps if budget_sweeps is not None else 1000
                traj_cap = 2 + (self.m + 1) * (sw + 1)
            tt = np.empty(traj_cap, np.float64)
            te = np.empty(traj_cap, np.float64)
            _check(lib().stmf_run(self._h, bs, secs, float(epsilon), _p(tt), _p(te), traj_cap, _p(counts)))
            L = int(counts[0])
            tt, te = tt[:L].copy(), te[:L].copy()
        keys = ("traj_len", "attempts", "accepts", "sweeps", "row_visits", "evaluated", "replicas",
                "product_passes")
        out = dict(zip(keys, (int(c) for c in counts)))
        if not self.sharded:
            rep = _i64()
            _check(lib().stmf_replayed_sweeps(self._h, ctypes.byref(rep)))
            out["replayed_sweeps_total"] = int(rep.value)
        return tt, te, out

    # diff-test hooks ------------------------------------------------------
    def set_max_attempts(self, cap: int):
        """Stop later runs after exactly `cap` attempts (0 = no cap): the checker's
        oracle.fit(max_attempts=...) on the device (host-driven sweep loop)."""
        _check(lib().stmf_set_max_attempts(self._h, int(cap)))

    def comm_info(self) -> dict:
        """Sharded sessions: the communicator's rank count and this rank (NCCL:
        ncclCommCount / ncclCommUserRank); kind "nccl", "local" or "none"."""
        out = np.zeros(3, np.int32)
        _check(lib().stmf_comm_info(self._h, _p(out)))
        return {"nranks": int(out[0]), "rank": int(out[1]),
                "kind": {1: "nccl", 0: "local", -1: "none"}[int(out[2])]}

    def set_audit(self, on: bool = True):
        """RunConfig.audit: after every sweep the caches are rebuilt and the objective
        recomputed from scratch; a mismatch raises StmfError code 7 (audit)."""
        _check(lib().stmf_set_audit(self._h, int(bool(on))))

    def product_given(self):
        P = np.empty(self.given, self.dtype)
        top2 = np.empty(self.given, self.dtype)
        arg = np.empty(self.given, np.int32)
        _check(lib().stmf_product_given(self._h, _p(P), _p(arg), _p(top2)))
        return P, arg, top2

    def col_scores(self):
        s = np.empty(self.n, np.float64)
        _check(lib().stmf_col_scores(self._h, _p(s)))
        return s

    def residuate(self, axis: int, vec):
        vec = np.ascontiguousarray(vec, dtype=self.dtype)
        out = np.empty(self.n if axis == 0 else self.m, self.dtype)
        _check(lib().stmf_residuate(self._h, axis, _p(vec), _p(out)))
        return out

    def try_update(self, op: int, i: int, j: int, k: int):
        u = np.empty(self.m, self.dtype)
        v = np.empty(self.n, self.dtype)
        f = _dbl()
        _check(lib().stmf_try_update(self._h, op, i, j, k, _p(u), _p(v), ctypes.byref(f)))
        return u, v, f.value

    def attempt(self, op: int, i: int, j: int, k: int):
        f = _dbl()
        acc = _int()
        _check(lib().stmf_attempt(self._h, op, i, j, k, ctypes.byref(f), ctypes.byref(acc)))
        return f.value, bool(acc.value)

    # other fit methods -------------------------------------------------------
    def set_strategy(self, family: int, selection: int = SEL_TD_A):
        _check(lib().stmf_set_strategy(self._h, int(family), int(selection)))

    def row_scores(self):
        s = np.empty(self.m, np.float64)
        _check(lib().stmf_row_scores(self._h, _p(s)))
        return s

    def matrix_candidates(self):
        rows = np.empty(self.given, np.int32)
        cols = np.empty(self.given, np.int32)
        ks = np.empty(self.given, np.int32)
        sc = np.empty(self.given, np.float64)
        _check(lib().stmf_matrix_candidates(self._h, _p(rows), _p(cols), _p(ks), _p(sc)))
        return rows, cols, ks, sc

    # measurement plumbing ----------------------------------------------------
    def stream_handle(self) -> int:
        h = _vp()
        _check(lib().stmf_stream(self._h, ctypes.byref(h)))
        return int(h.value or 0)

    def set_profiling(self, on: bool = True):
        _check(lib().stmf_set_profiling(self._h, int(on)))

    def counters(self) -> dict:
        c = np.zeros(8, np.int64)
        _check(lib().stmf_counters(self._h, _p(c)))
        keys = ("launches", "cub_sorts", "phaseB_launches", "phaseB_ns", "phaseB_timed",
                "product_passes", "replicas", "given")
        return dict(zip(keys, (int(x) for x in c)))

    def bench_product(self, reps: int = 10, flush_l2: bool = True):
        ms = _dbl()
        err = _dbl()
        _check(lib().stmf_bench_product(self._h, reps, int(flush_l2), ctypes.byref(ms), ctypes.byref(err)))
        return ms.value, err.value


def masked_rmse(pred, truth, mask, device: int | None = None) -> float:
    pred = np.ascontiguousarray(pred, dtype=np.float64)
    truth = np.ascontiguousarray(truth, dtype=np.float64)
    mask = np.ascontiguousarray(mask, dtype=bool)
    if pred.shape != truth.shape or mask.shape != pred.shape or pred.ndim != 2:
        raise ValueError("pred, truth and mask must be 2-d arrays of one shape")
    out = _dbl()
    dev = default_device() if device is None else device
    _check(lib().stmf_masked_rmse(pred.shape[0], pred.shape[1], _p(pred), _p(truth), _p(mask.view(np.uint8)), dev,
                                  ctypes.byref(out)))
    return out.value


def distance_correlation(x, y, device: int | None = None) -> float:
    x = np.ascontiguousarray(x, dtype=np.float64).ravel()
    y = np.ascontiguousarray(y, dtype=np.float64).ravel()
    out = _dbl()
    dev = default_device() if device is None else device
    _check(lib().stmf_distance_correlation(x.size, _p(x), _p(y), dev, ctypes.byref(out)))
    return out.value


def csv_read(path: str, has_header: bool = False, threads: int = 0):
    """Native load_matrix_csv: (values float64 with NaN where missing, mask bool)."""
    m, n, h = _i64(), _i64(), _vp()
    _check(lib().stmf_csv_open(os.fsencode(path), int(has_header), ctypes.byref(h), ctypes.byref(m),
                               ctypes.byref(n)))
    try:
        values = np.empty((m.value, n.value), np.float64)
        mask = np.empty((m.value, n.value), np.uint8)
        _check(lib().stmf_csv_fill(h, _p(values), _p(mask), int(threads)))
    finally:
        lib().stmf_csv_close(h)
    return values, mask.view(bool)


def release_memory(device: int | None = None):
    """Return the device memory pool's unused blocks (kept for reuse by later sessions)."""
    _check(lib().stmf_release_memory(default_device() if device is None else device))


def b_norm(values, device: int | None = None) -> float:
    v = np.ascontiguousarray(values, dtype=np.float64).ravel()
    out = _dbl()
    _check(lib().stmf_b_norm(v.size, _p(v), default_device() if device is None else device, ctypes.byref(out)))
    return out.value
