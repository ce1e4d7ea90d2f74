"""Golden fixture for the binary64 path on config 2's data distribution
(log2(1 + lognormal), 50% missing, rank 5): the UNMODIFIED reference's fast_stmf on a
200 x 400 crop of config 2 for 5 sweeps (tests/golden/c2crop.npz).  Run in the build
container: python tests/golden/make_golden_c2crop.py"""
import os
import sys
import time

import numpy as np

REF = os.environ.get("STMF_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import tropfact  # noqa: E402
from tropfact import engine  # noqa: E402

from paper_2205_06619_b200 import gen  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def main():
    C = gen.config2()
    vals, mask = C.values[:200, :400], C.mask[:200, :400]
    R = tropfact.MaskedMatrix(np.where(mask, vals, np.nan), mask)
    cfg = engine.RunConfig(rank=5, budget_sweeps=5, epsilon=0.0, seed=42)
    t = time.time()
    pair, traj = tropfact.fast_stmf(R, 5, cfg)
    print(f"reference fit: {time.time() - t:.1f} s, {len(traj.errors)} samples, "
          f"{traj.errors[0]:.6f} -> {traj.errors[-1]:.6f}")
    np.savez_compressed(os.path.join(HERE, "c2crop.npz"), R=vals, M=mask, U=pair.U, V=pair.V,
                        traj_t=np.array(traj.times), traj_e=np.array(traj.errors), rank=np.int64(5),
                        sweeps=np.int64(5), seed=np.int64(42))


if __name__ == "__main__":
    main()
