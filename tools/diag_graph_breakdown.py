"""Diagnostics: sweep-graph time breakdown (phase B / escalation rounds / accept path)
from the device ticks (STMF_GRAPH_STATS=1 prints it per sweep).
    STMF_GRAPH_STATS=1 python tools/diag_graph_breakdown.py CONFIG WARM SWEEPS"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2205_06619_b200 import _ext, engine, gen  # noqa: E402

cfg, warm, sweeps = (int(x) for x in sys.argv[1:4])
C = gen.CONFIGS[cfg]
R = C["make"]()
rng = np.random.default_rng(42)
work, _ = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, C["rank"], 5, rng)
s = _ext.Session(work.values, work.mask, C["rank"])
s.set_factors(U0)
s.run(budget_sweeps=warm, epsilon=0.0)
s.set_profiling(True)
for k in range(sweeps):
    t = time.time()
    tt, te, cnt = s.run(budget_sweeps=1, epsilon=0.0)
    print(f"sweep {warm + k + 1}: {1e3 * (time.time() - t):.1f} ms wall", cnt, flush=True)
