"""Diagnostics: wall time of each part of one fast_stmf call (config 2, K sweeps)."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_06619_b200 as pkg  # noqa: E402
from paper_2205_06619_b200 import engine, gen  # noqa: E402

K = int(sys.argv[1]) if len(sys.argv) > 1 else 5
R = gen.config2()
pkg.fast_stmf(R, 5, pkg.RunConfig(rank=5, budget_sweeps=1, epsilon=0.0, seed=1))  # warm context
for rep in range(2):
    T = {}
    t = time.perf_counter()
    rng = np.random.default_rng(42)
    work, ori = engine._orient_faststmf(R, rng)
    T["orient"] = time.perf_counter() - t; t = time.perf_counter()
    U0 = engine.acol_means(work, 5, 5, rng)
    T["acol_means"] = time.perf_counter() - t; t = time.perf_counter()
    s = engine.FitSession(work, 5)
    T["session"] = time.perf_counter() - t; t = time.perf_counter()
    s.set_factors(U0)
    T["set_factors"] = time.perf_counter() - t; t = time.perf_counter()
    tt, te, cnt = s.run(K, None, 0.0)
    T["run"] = time.perf_counter() - t; t = time.perf_counter()
    U, V = s.get_factors()
    s.close()
    T["get+close"] = time.perf_counter() - t
    t = time.perf_counter()
    pkg.fast_stmf(R, 5, pkg.RunConfig(rank=5, budget_sweeps=K, epsilon=0.0, seed=42))
    T["fast_stmf_total"] = time.perf_counter() - t
    print({k: round(v * 1e3, 1) for k, v in T.items()}, cnt["attempts"], flush=True)
