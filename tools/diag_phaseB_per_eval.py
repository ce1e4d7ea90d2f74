"""Diagnostics: phase-B device time per evaluation over the first two config-2 sweeps (host loop, profiled launches)."""
import os, sys, time, numpy as np
sys.path.insert(0, "/root/repo")
from paper_2205_06619_b200 import gen, engine, _ext
R = gen.config2()
rng = np.random.default_rng(42)
work, ori = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, 5, 5, rng)
s = _ext.Session(work.values, work.mask, 5); s.set_factors(U0)
s.set_profiling(True)
c0 = s.counters()
tt, te, cnt = s.run(budget_sweeps=2, epsilon=0.0)
c1 = s.counters()
ns = c1["phaseB_ns"] - c0["phaseB_ns"]; nl = c1["phaseB_timed"] - c0["phaseB_timed"]
print(os.environ.get("STMF_LIB", "base"), "evaluated", cnt["evaluated"], "phaseB ms", ns / 1e6, "us/eval", ns / 1e3 / cnt["evaluated"], "launches", nl)
