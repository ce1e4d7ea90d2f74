"""Diagnostics: row visits/s and profiled phase-B time per evaluation for a config
over a wall-clock budget (host-driven loop): python tools/diag_phaseB_cfg.py CONFIG SECONDS"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_06619_b200 import _ext, engine, gen  # noqa: E402

cfg, secs = int(sys.argv[1]), float(sys.argv[2])
C = gen.CONFIGS[cfg]
R = C["make"]()
rng = np.random.default_rng(42)
work, _ = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, C["rank"], 5, rng)
for lib in (os.environ.get("LIBS") or os.environ.get("STMF_LIB", "")).split(","):
    if lib:
        os.environ["STMF_LIB"] = lib
        _ext._lib = None
    s = _ext.Session(work.values, work.mask, C["rank"])
    s.set_factors(U0)
    s.set_profiling(True)
    c0 = s.counters()
    t = time.time()
    tt, te, cnt = s.run(budget_seconds=secs, epsilon=0.0)
    dt = time.time() - t
    c1 = s.counters()
    ns = c1["phaseB_ns"] - c0["phaseB_ns"]
    nl = c1["phaseB_timed"] - c0["phaseB_timed"]
    print(f"{lib or 'default'} cfg {cfg}: row visits/s {cnt['row_visits'] / dt:.1f} evaluated {cnt['evaluated']} "
          f"phaseB {ns / 1e6:.1f} ms / {nl} launches = {ns / 1e3 / max(nl, 1):.1f} us, "
          f"{ns / max(cnt['evaluated'], 1):.1f} ns/eval, err {te[-1]:.6f}", flush=True)
    s.close()
