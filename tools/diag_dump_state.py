"""Diagnostics: dump the work-orientation data and factors after N sweeps to gpurun_out/state_cN.npz."""
import sys, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
from paper_2205_06619_b200 import gen, engine, _ext
cfg = int(sys.argv[1]); sweeps = float(sys.argv[2])
C = gen.CONFIGS[cfg]; R = C["make"]()
rng = np.random.default_rng(42)
work, ori = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, C["rank"], 5, rng)
s = _ext.Session(work.values, work.mask, C["rank"]); s.set_factors(U0)
if sweeps >= 1:
    s.run(budget_sweeps=int(sweeps), epsilon=0.0)
else:
    s.run(budget_seconds=sweeps * 100, epsilon=0.0)
U, V = s.get_factors()
np.savez_compressed(f"gpurun_out/state_c{cfg}.npz", X=work.values, M=work.mask, U=U, V=V)
