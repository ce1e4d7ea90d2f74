"""Golden fixtures for every fit method of the reference (tests/golden/strategies.npz),
generated from the UNMODIFIED reference package (tropfact, read-only import from
/root/reference/pkg/src).  Run in the build container:
    python tests/golden/make_golden_strategies.py

Each case is ``tropfact.fit(R, rank, method, RunConfig(...))`` (strategies.py:351-357;
STMF -> engine.stmf_baseline, engine.py:383-385) on a small seeded matrix: the original
R and mask, the method name, the config and the resulting factors and trajectory.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

REF = os.environ.get("STMF_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import tropfact  # noqa: E402
from tropfact import datagen, engine, tropical  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

METHODS = ["STMF", "STMF_ByElement_PermC_TD", "STMF_ByElement_PermC_TD_W",
           "STMF_ByMatrix_NoPerm_TD", "STMF_ByMatrix_NoPerm_TD_W"]
for perm in ("NoPerm", "PermR", "RandPermR"):
    for sel in ("TD", "TD_A", "TD_B", "SEQ"):
        for w in ("", "_W"):
            METHODS.append(f"STMF_ByRow_{perm}_{sel}{w}")


def data(rng, m, n, r, frac):
    A = rng.random((m, r))
    B = rng.random((r, n))
    X = tropical.trop_matmul(A, B) + rng.normal(0, 0.05, (m, n))
    R, _ = datagen.apply_mask(X, frac, seed=int(rng.integers(1 << 30)))
    return R


def main():
    rng = np.random.default_rng(11)
    shapes = [("tall", 14, 9, 2, 0.25, 3), ("wide", 8, 13, 3, 0.2, 3), ("med", 36, 24, 3, 0.3, 3)]
    out = {}
    names = []
    for tag, m, n, r, frac, sweeps in shapes:
        R = data(rng, m, n, r, frac)
        for meth in METHODS:
            # ByMatrix makes one update per sweep: give it more sweeps
            sw = sweeps * 4 if "ByMatrix" in meth else sweeps
            cfg = engine.RunConfig(rank=r, budget_sweeps=sw, epsilon=0.0, seed=31)
            t0 = time.time()
            pair, traj = tropfact.fit(R, r, meth, cfg)
            name = f"{tag}_{meth}"
            names.append(name)
            out.update({f"{name}|U": pair.U, f"{name}|V": pair.V, f"{name}|traj_t": np.array(traj.times),
                        f"{name}|traj_e": np.array(traj.errors)})
            print(f"{name}: {len(traj.errors)} samples {traj.errors[0]:.6f} -> {traj.errors[-1]:.6f} "
                  f"({time.time() - t0:.1f}s)", flush=True)
        out[f"{tag}|R"] = R.values
        out[f"{tag}|M"] = R.mask
        out[f"{tag}|rank"] = np.int64(r)
        out[f"{tag}|sweeps"] = np.int64(sweeps)
    out["names"] = np.array(names)
    out["seed"] = np.int64(31)
    np.savez_compressed(os.path.join(HERE, "strategies.npz"), **out)


if __name__ == "__main__":
    main()
