"""Diagnostics: wall time of config 1's full 100-sweep fit through fast_stmf, with
fixpoint-sweep replay on (default) and off (STMF_FIXPOINT_REPLAY=0)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2205_06619_b200 as pkg  # noqa: E402
from paper_2205_06619_b200 import gen  # noqa: E402

R = gen.config1()
cfg = pkg.RunConfig(rank=3, budget_sweeps=100, epsilon=0.0, seed=42)
pkg.fast_stmf(R, 3, pkg.RunConfig(rank=3, budget_sweeps=1, epsilon=0.0, seed=1))
for replay in ("1", "0", "1", "0"):
    os.environ["STMF_FIXPOINT_REPLAY"] = replay
    t = time.perf_counter()
    pair, traj = pkg.fast_stmf(R, 3, cfg)
    print(f"replay={replay}: {time.perf_counter() - t:.3f} s, final {traj.final_error!r}, "
          f"replayed {traj.counts['replayed_sweeps_total']}", flush=True)
