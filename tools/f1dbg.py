import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
os.environ["STMF_GRAPH"]="0"; os.environ["STMF_FAST1_CHECK"]="1"
import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import _ext, engine, gen
R = gen.config2(); R = pkg.MaskedMatrix(R.values[:200,:400], R.mask[:200,:400])
rng = np.random.default_rng(42)
work, _ = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, 5, 5, rng)
with _ext.Session(work.values, work.mask, 5) as s:
    s.set_factors(U0)
    tt, te, c = s.run(budget_sweeps=2, epsilon=0.0)
print(c)
