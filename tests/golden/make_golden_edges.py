"""Edge-shape golden fixtures (tests/golden/edges.npz) from the UNMODIFIED reference:
single rows / columns, tiny fully-given matrices, rank above min(m, n), ties from
quantised data, for FastSTMF and the other methods.  Run in the build container:
    python tests/golden/make_golden_edges.py"""
import os
import sys

import numpy as np

REF = os.environ.get("STMF_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import tropfact  # noqa: E402
from tropfact import datagen, engine, tropical  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
METHODS = ["FastSTMF", "STMF", "STMF_ByElement_PermC_TD", "STMF_ByMatrix_NoPerm_TD_W", "STMF_ByRow_PermR_SEQ_W",
           "STMF_ByRow_NoPerm_TD_B"]


def main():
    rng = np.random.default_rng(99)
    cases = {}
    cases["row1"] = (rng.random((1, 7)) * 3, np.ones((1, 7), bool), 2)
    cases["col1"] = (rng.random((6, 1)) * 3, np.ones((6, 1), bool), 1)
    cases["full2x2"] = (rng.random((2, 2)), np.ones((2, 2), bool), 2)
    X = rng.random((3, 4))
    cases["rank_gt"] = (X, np.ones((3, 4), bool), 5)
    Q = np.round(rng.random((9, 11)) * 4) / 4  # many exact ties
    R, _ = datagen.apply_mask(Q, 0.3, seed=5)
    cases["ties"] = (Q, R.mask, 3)
    A = rng.random((12, 2))
    B = rng.random((2, 10))
    Xm = tropical.trop_matmul(A, B)  # exact max-plus data: zero-error optimum reachable
    cases["exact"] = (Xm, np.ones((12, 10), bool), 2)
    out, names = {}, []
    for tag, (X, M, r) in cases.items():
        R = tropical.MaskedMatrix(np.where(M, X, np.nan), M)
        out[f"{tag}|X"] = X
        out[f"{tag}|M"] = M
        out[f"{tag}|rank"] = np.int64(r)
        for meth in METHODS:
            sweeps = 8 if "ByMatrix" in meth else 3
            cfg = engine.RunConfig(rank=r, budget_sweeps=sweeps, epsilon=0.0, seed=7)
            pair, traj = tropfact.fit(R, r, meth, cfg)
            name = f"{tag}|{meth}"
            names.append(name)
            out[f"{name}|U"] = pair.U
            out[f"{name}|V"] = pair.V
            out[f"{name}|traj_t"] = np.array(traj.times)
            out[f"{name}|traj_e"] = np.array(traj.errors)
            out[f"{name}|sweeps"] = np.int64(sweeps)
            print(name, len(traj.errors), traj.errors[0], traj.errors[-1], flush=True)
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "edges.npz"), **out)


if __name__ == "__main__":
    main()
