"""Diagnostics: one wall-clock-budgeted run after warm sweeps, for ncu captures (python tools/diag_budget_run.py CONFIG SECONDS WARM)."""
import sys, time, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2205_06619_b200 import gen, engine, _ext
cfgno = int(sys.argv[1]); secs = float(sys.argv[2]); warm = int(sys.argv[3]) if len(sys.argv) > 3 else 0
C = gen.CONFIGS[cfgno]
R = C["make"]()
rng = np.random.default_rng(42)
work, ori = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, C["rank"], 5, rng)
s = _ext.Session(work.values, work.mask, C["rank"]); s.set_factors(U0)
for _ in range(warm):
    s.run(budget_sweeps=1, epsilon=0.0)
t = time.time()
tt, te, cnt = s.run(budget_seconds=secs, epsilon=0.0)
print(f"{(time.time()-t)*1e3:.1f} ms", cnt, s.counters(), flush=True)
