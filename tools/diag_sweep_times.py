"""Diagnostics: per-sweep wall times of the device engine on a config (python tools/diag_sweep_times.py CONFIG SWEEPS)."""
import sys, time, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import gen, engine, _ext
cfgno = int(sys.argv[1]) if len(sys.argv) > 1 else 2
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
C = gen.CONFIGS[cfgno]
t = time.time(); R = C["make"](); print("gen", time.time() - t, flush=True)
rng = np.random.default_rng(42)
work, ori = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, C["rank"], 5, rng)
t = time.time()
s = _ext.Session(work.values, work.mask, C["rank"]); s.set_factors(U0)
print("session", time.time() - t, "given", s.given, flush=True)
for sw in range(sweeps):
    c0 = s.counters()
    t = time.time()
    tt, te, cnt = s.run(budget_sweeps=1, epsilon=0.0)
    dt = time.time() - t
    c1 = s.counters()
    d = {k: c1[k] - c0[k] for k in c1}
    print(f"sweep {sw+1}: {dt*1e3:.1f} ms err {te[0]:.6f}->{te[-1]:.6f} {cnt} delta {d}", flush=True)
