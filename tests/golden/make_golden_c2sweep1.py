"""Golden fixture of BASELINE.json configs[1] itself (config 2: 500 x 1000 work shape,
rank 5, fp64): the UNMODIFIED reference's fast_stmf for 1 sweep (~20 min of numpy), seeds
as in SURVEY.md §8d (data 0, mask 1, fit 42).  Stores the trajectory and the factors.
    python tests/golden/make_golden_c2sweep1.py"""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.environ.get("STMF_REFERENCE", "/root/reference/pkg/src"))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tropfact  # noqa: E402
from tropfact import engine  # noqa: E402

from paper_2205_06619_b200 import gen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
C = gen.config2()
R = tropfact.MaskedMatrix(np.where(C.mask, C.values, np.nan), C.mask)
cfg = engine.RunConfig(rank=5, budget_sweeps=1, epsilon=0.0, seed=42)
t = time.time()
pair, traj = tropfact.fast_stmf(R, 5, cfg)
print(f"reference: {time.time() - t:.0f} s, {len(traj.errors)} samples, {traj.errors[0]!r} -> {traj.errors[-1]!r}")
np.savez_compressed(os.path.join(HERE, "c2sweep1.npz"), U=pair.U, V=pair.V, traj_t=np.array(traj.times),
                    traj_e=np.array(traj.errors))
