"""Device fit of configs 1, 2 and 3 from the seeded init (fit seed 42, as fast_stmf):
saves the state after sweep 1 (work orientation) to tests/golden/c{C}_state_s1.npz,
the common starting state of bench.py's timed window, of its end-to-end leg and of
the reference arm's sample (bench.py docstring), and prints per-sweep timings of
sweeps 1..S.  The bench re-derives this state in its warm-up and checks it bitwise.

    python tools/make_states.py [S]
"""
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("STMF_FIXPOINT_REPLAY", "0")
from paper_2205_06619_b200 import _ext, engine, gen  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 3
for cfg in (1, 2, 3):
    C = gen.CONFIGS[cfg]
    R = C["make"]()
    rng = np.random.default_rng(42)
    work, _ = engine._orient_faststmf(R, rng)
    U0 = engine.acol_means(work, C["rank"], 5, rng)
    N = int(work.mask.sum())
    with _ext.Session(work.values, work.mask, C["rank"]) as s:
        s.set_factors(U0)
        for sw in range(1, S + 1):
            t = time.perf_counter()
            tt, te, c = s.run(budget_sweeps=1, epsilon=0.0)
            dt = time.perf_counter() - t
            print(f"config {cfg} sweep {sw}: {dt:.3f} s attempts {c['attempts']} accepts {c['accepts']} "
                  f"evaluated {c['evaluated']} err {te[-1]!r} Gentries/s {c['attempts'] * N / dt / 1e9:.1f}",
                  flush=True)
            if sw == 1:
                U, V = s.get_factors()
                np.savez_compressed(os.path.join(ROOT, "tests", "golden", f"c{cfg}_state_s1.npz"), U=U, V=V,
                                    err=np.array(te[-1]), sweeps=np.array(1), attempts=np.array(c["attempts"]))
