import sys, time, numpy as np
sys.path.insert(0, '.')
from paper_2205_06619_b200 import gen, engine, _ext
m = int(sys.argv[1]) if len(sys.argv) > 1 else 32768
R = gen.config4(m=m, n=m, blocks=max(1, m // 512))
rng = np.random.default_rng(42)
work, _ = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, 20, 5, rng)
s = _ext.Session(work.values, work.mask, 20); s.set_factors(U0)
t = time.time()
tt, te, c = s.run(budget_seconds=float(sys.argv[2]) if len(sys.argv) > 2 else 3.0, epsilon=0.0)
print(time.time() - t, c)
