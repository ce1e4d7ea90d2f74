import sys, time, numpy as np
sys.path.insert(0, '.')
import torch
import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import gen, engine, _ext
C = gen.CONFIGS[2]; R = C["make"]()
torch.cuda.synchronize()
for rep in range(3):
    t0 = time.perf_counter()
    rng = np.random.default_rng(42)
    work, ori = engine._orient_faststmf(R, rng)
    U0 = engine.acol_means(work, C["rank"], 5, rng)
    t1 = time.perf_counter()
    s = _ext.Session(work.values, work.mask, C["rank"])
    t2 = time.perf_counter()
    s.set_factors(U0)
    t3 = time.perf_counter()
    tt, te, cnt = s.run(budget_sweeps=5, epsilon=0.0)
    t4 = time.perf_counter()
    U, V = s.get_factors()
    s.close()
    t5 = time.perf_counter()
    print(f"host prep {t1-t0:.3f} session {t2-t1:.3f} set_factors {t3-t2:.3f} run5 {t4-t3:.3f} get+close {t5-t4:.3f}", flush=True)
    t0 = time.perf_counter()
    pair, traj = pkg.fast_stmf(R, C["rank"], pkg.RunConfig(rank=C["rank"], budget_sweeps=5, epsilon=0.0, seed=42))
    print(f"fast_stmf {time.perf_counter()-t0:.3f}", flush=True)
