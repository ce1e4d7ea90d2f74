"""Diagnostics: wall time of each part of one fast_stmf(..., budget_sweeps=1, init=S1) call at
config 3 (the bench's e2e step): host orientation, session creation (H2D + compaction),
factor upload + caches, the sweep, read-back.

    python tools/diag_e2e_c3.py [REPS]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("STMF_FIXPOINT_REPLAY", "0")
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2205_06619_b200 as pkg  # noqa: E402
from paper_2205_06619_b200 import engine  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 2
C, R, work0, ori0, U0, (U1, V1) = bench.workload(3)
r = C["rank"]
Uo, Vo = ori0.restore(U1, V1)
cfg = pkg.RunConfig(rank=r, budget_sweeps=1, epsilon=0.0, seed=42)
pkg.fast_stmf(R, r, cfg, init=(Uo, Vo))  # warm context and pools
for rep in range(reps):
    T = {}
    t = time.perf_counter()
    R.validate_coverage()
    rng = np.random.default_rng(42)
    work, ori = engine._orient_faststmf(R, rng)
    T["validate+orient"] = time.perf_counter() - t; t = time.perf_counter()
    Ui, Vi = ori.apply_factors(np.asarray(Uo, dtype=R.dtype), np.asarray(Vo, dtype=R.dtype))
    T["apply_factors"] = time.perf_counter() - t; t = time.perf_counter()
    s = engine.FitSession(work, r)
    torch.cuda.synchronize()
    T["session"] = time.perf_counter() - t; t = time.perf_counter()
    s.set_factors(Ui, Vi)
    torch.cuda.synchronize()
    T["set_factors"] = time.perf_counter() - t; t = time.perf_counter()
    tt, te, cnt = s.run(1, None, 0.0)
    T["run"] = time.perf_counter() - t; t = time.perf_counter()
    U, V = s.get_factors()
    s.close()
    T["get+close"] = time.perf_counter() - t; t = time.perf_counter()
    ori.restore(U, V)
    T["restore"] = time.perf_counter() - t
    t = time.perf_counter()
    pkg.fast_stmf(R, r, cfg, init=(Uo, Vo))
    torch.cuda.synchronize()
    T["fast_stmf_total"] = time.perf_counter() - t
    print({k: round(v * 1e3, 1) for k, v in T.items()}, cnt["attempts"], flush=True)
