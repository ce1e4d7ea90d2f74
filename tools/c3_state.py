"""Device run of config 3 from the seeded init (fit seed 42): times each of the first
S sweeps and saves the state after sweep `save_at` (work orientation) to
tests/golden/c3_state_s3.npz -- the common starting state of bench.py's timed window
and of the reference arm's sample (bench.py docstring)."""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("STMF_FIXPOINT_REPLAY", "0")
from paper_2205_06619_b200 import _ext, engine, gen  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 5
save_at = 3
R = gen.config3()
rng = np.random.default_rng(42)
work, _ = engine._orient_faststmf(R, rng)
U0 = engine.acol_means(work, 10, 5, rng)
with _ext.Session(work.values, work.mask, 10) as s:
    s.set_factors(U0)
    for sw in range(1, S + 1):
        t = time.perf_counter()
        tt, te, c = s.run(budget_sweeps=1, epsilon=0.0)
        dt = time.perf_counter() - t
        print(f"sweep {sw}: {dt:.2f} s attempts {c['attempts']} accepts {c['accepts']} evaluated {c['evaluated']} "
              f"err {te[-1]!r} Gentries/s {c['attempts'] * int(work.mask.sum()) / dt / 1e9:.1f}", flush=True)
        if sw == save_at:
            U, V = s.get_factors()
            np.savez_compressed(os.path.join(ROOT, "tests", "golden", "c3_state_s3.npz"), U=U, V=V,
                                err=np.array(te[-1]), sweeps=np.array(save_at))
