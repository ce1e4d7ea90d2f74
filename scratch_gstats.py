import sys, numpy as np
sys.path.insert(0, '.')
from paper_2205_06619_b200 import gen, engine, _ext
cfg = int(sys.argv[1]); sweeps = int(sys.argv[2])
C = gen.CONFIGS[cfg]; R = C["make"]()
rng = np.random.default_rng(42)
work, ori = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, C["rank"], 5, rng)
s = _ext.Session(work.values, work.mask, C["rank"]); s.set_factors(U0)
s.set_profiling(True)
for _ in range(sweeps): s.run(budget_sweeps=1, epsilon=0.0)
