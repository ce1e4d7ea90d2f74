import sys, time, json, os, numpy as np
sys.path.insert(0, '.')
import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import gen, engine, _ext
cfg = int(sys.argv[1]); sweeps = int(sys.argv[2])
C = gen.CONFIGS[cfg]; R = C["make"]()
rng = np.random.default_rng(42)
work, ori = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, C["rank"], 5, rng)
s = _ext.Session(work.values, work.mask, C["rank"]); s.set_factors(U0)
s.objective()
import torch; torch.cuda.synchronize()
t = time.perf_counter()
tt, te, cnt = s.run(budget_sweeps=sweeps, epsilon=0.0)
dt = time.perf_counter() - t
print(json.dumps({"config": cfg, "graph": os.environ.get("STMF_GRAPH", "1"), "sweeps": sweeps, "seconds": dt,
                  "final": te[-1], "attempts": cnt["attempts"], "row_visits": cnt["row_visits"],
                  "evaluated": cnt["evaluated"]}), flush=True)
