"""Diagnostics: launch-count / timing probe of one fit (kept from round-1 investigations)."""
import sys, numpy as np, torch
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2205_06619_b200 import gen, engine, _ext
cfg = int(sys.argv[1]); warm = int(sys.argv[2]); secs = float(sys.argv[3]) if len(sys.argv) > 3 else 0
C = gen.CONFIGS[cfg]; R = C["make"]()
rng = np.random.default_rng(42)
work, ori = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, C["rank"], 5, rng)
s = _ext.Session(work.values, work.mask, C["rank"]); s.set_factors(U0)
if warm: s.run(budget_sweeps=warm, epsilon=0.0)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
if secs: print(s.run(budget_seconds=secs, epsilon=0.0)[2])
else: print(s.run(budget_sweeps=1, epsilon=0.0)[2])
torch.cuda.cudart().cudaProfilerStop()
