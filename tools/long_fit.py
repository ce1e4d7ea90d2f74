"""Long fit record: config C from the seeded init (fit seed 42, as fast_stmf), sweep by
sweep on one device until S sweeps or T seconds, every sweep executed (no fixpoint
replay).  One JSON line per sweep: time, attempts, accepts, evaluated, error.

    python tools/long_fit.py C S T out.jsonl [start.npz FIRST_SWEEP]

With start.npz (U, V of the work orientation, e.g. the _factors.npz of an earlier run)
the fit continues from that state, numbering sweeps from FIRST_SWEEP.
"""
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ["STMF_FIXPOINT_REPLAY"] = "0"
from paper_2205_06619_b200 import _ext, engine, gen  # noqa: E402

cfg, S, T, out = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3]), sys.argv[4]
start = np.load(sys.argv[5]) if len(sys.argv) > 5 else None
first = int(sys.argv[6]) if len(sys.argv) > 6 else 1
C = gen.CONFIGS[cfg]
t0 = time.time()
R = C["make"]()
rng = np.random.default_rng(42)
work, _ = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, C["rank"], 5, rng)
N = int(work.mask.sum())
tgen = time.time() - t0
with open(out, "w") as f, _ext.Session(work.values, work.mask, C["rank"]) as s:
    if start is None:
        s.set_factors(U0)
    else:
        s.set_factors(start["U"].astype(work.dtype), start["V"].astype(work.dtype))
    f.write(json.dumps({"config": cfg, "shape": list(work.shape), "rank": C["rank"], "given": N,
                        "init_error": s.objective(), "gen_s": tgen, "first_sweep": first}) + "\n")
    t_start = time.time()
    for sw in range(first, S + 1):
        t = time.perf_counter()
        tt, te, c = s.run(budget_sweeps=1, epsilon=0.0)
        dt = time.perf_counter() - t
        rec = {"sweep": sw, "seconds": dt, "attempts": c["attempts"], "accepts": c["accepts"],
               "evaluated": c["evaluated"], "row_visits": c["row_visits"], "error": te[-1],
               "gentries_per_s": c["attempts"] * N / dt / 1e9}
        f.write(json.dumps(rec) + "\n")
        f.flush()
        print(json.dumps(rec), flush=True)
        if c["accepts"] == 0:
            f.write(json.dumps({"fixpoint_at_sweep": sw}) + "\n")
            break
        if time.time() - t_start > T:
            break
    U, V = s.get_factors()
    np.savez_compressed(out.replace(".jsonl", "_factors.npz"), U=U, V=V)
