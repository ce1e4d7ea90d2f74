import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import gen, engine, _ext
C = gen.CONFIGS[2]; R = C["make"]()
rng = np.random.default_rng(42)
work, ori = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, C["rank"], 5, rng)
s = _ext.Session(work.values, work.mask, C["rank"]); s.set_factors(U0)
if len(sys.argv) > 1: s.set_profiling(True)
for _ in range(8): s.run(budget_sweeps=1, epsilon=0.0)
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.perf_counter()
    pair, traj = pkg.fast_stmf(R, C["rank"], pkg.RunConfig(rank=C["rank"], budget_sweeps=5, epsilon=0.0, seed=42))
    torch.cuda.synchronize()
    print(f"fast_stmf {time.perf_counter()-t0:.3f}", flush=True)
