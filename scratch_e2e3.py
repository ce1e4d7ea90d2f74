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
s.set_profiling(True)
for _ in range(8): s.run(budget_sweeps=1, epsilon=0.0)
torch.cuda.synchronize()
for rep in range(4):
    T = [time.perf_counter()]
    rng = np.random.default_rng(42)
    w2, o2 = engine._orient_faststmf(R, rng); U2 = engine.acol_means(w2, C["rank"], 5, rng); T.append(time.perf_counter())
    fs = engine.FitSession(w2, C["rank"], 0); T.append(time.perf_counter())
    fs.__enter__(); fs.set_factors(U2); T.append(time.perf_counter())
    tt, te, cnt = fs.run(5, None, 0.0); T.append(time.perf_counter())
    U, V = fs.get_factors(); T.append(time.perf_counter())
    fs.__exit__(None, None, None); T.append(time.perf_counter())
    print("prep %.3f create %.3f setf %.3f run %.3f get %.3f close %.3f" % tuple(T[i+1]-T[i] for i in range(6)), flush=True)
