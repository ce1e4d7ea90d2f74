"""Generate the golden fixtures under tests/golden/ from the UNMODIFIED reference
package (tropfact, imported read-only from /root/reference/pkg/src).

Run in the build container (the GPU box has no /root/reference):
    python tests/golden/make_golden.py
Outputs (all small, committed):
  ops.npz        random-instance outputs of trop_matmul / argmax_grid / td_grid
                 column sums / _residuate_row / _residuate_col / approx_error /
                 f_ulf / f_urf / b_norm (pairwise-sum facts)
  fits.npz       fast_stmf runs (original R, mask, seed, budget) with the work-
                 orientation data, the Random-Acol factors, the final factors and the
                 full trajectory
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("STMF_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
import tropfact  # noqa: E402
from tropfact import datagen, engine, strategies, tropical  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def rand_masked(rng, m, n, frac):
    X = rng.random((m, n)) * 3.0 - 0.5
    R, _ = datagen.apply_mask(X, frac, seed=rng)
    return R


def make_ops():
    rng = np.random.default_rng(2024)
    out = {}
    cases = []
    for c in range(40):
        m = int(rng.integers(1, 14))
        n = int(rng.integers(1, 14))
        r = int(rng.integers(1, 5))
        frac = float(rng.choice([0.0, 0.2, 0.5]))
        if m * n - int(np.floor(frac * m * n)) < max(m, n):
            frac = 0.0
        R = rand_masked(rng, m, n, frac)
        U = rng.random((m, r)) * 2.0
        V = rng.random((r, n)) * 2.0
        if c % 5 == 0:  # ties in the max-plus argmax
            U = np.round(U * 4) / 4
            V = np.round(V * 4) / 4
        P = tropical.trop_matmul(U, V)
        arg = tropical.argmax_grid(U, V)
        scores = tropical.td_grid(R, U, V).sum(axis=0)
        u = rng.random(m)
        v = rng.random(n)
        rr = engine._residuate_row(R, u)
        rc = engine._residuate_col(R, v)
        err = tropical.approx_error(R, U, V)
        # one F-ULF / F-URF outcome at a random given position
        gi, gj = np.nonzero(R.mask)
        t = int(rng.integers(0, gi.size))
        i, j, k = int(gi[t]), int(gj[t]), int(rng.integers(0, r))
        U1, V1 = U.copy(), V.copy()
        o1 = engine.f_ulf(R, U1, V1, i, j, k)
        U2, V2 = U.copy(), V.copy()
        o2 = engine.f_urf(R, U2, V2, i, j, k)
        pre = f"c{c}_"
        out.update({pre + "X": R.values, pre + "M": R.mask, pre + "U": U, pre + "V": V,
                    pre + "P": P, pre + "arg": arg, pre + "scores": scores, pre + "u": u,
                    pre + "v": v, pre + "rr": rr, pre + "rc": rc, pre + "err": np.float64(err),
                    pre + "ijk": np.array([i, j, k]), pre + "ulf_U": U1, pre + "ulf_V": V1,
                    pre + "ulf_f": np.float64(o1.f), pre + "urf_U": U2, pre + "urf_V": V2,
                    pre + "urf_f": np.float64(o2.f)})
        cases.append(c)
    # numpy pairwise-summation facts (b_norm = np.sum(np.sort(|w|)))
    sums = []
    for t in range(30):
        n = int(rng.integers(1, 3000)) if t < 27 else int(rng.integers(50_000, 200_000))
        w = rng.normal(size=n) * rng.random(n) ** 6
        out[f"bn{t}_w"] = w
        sums.append(tropical.b_norm(w))
    out["bn_sums"] = np.array(sums)
    out["n_ops"] = np.int64(len(cases))
    out["n_bn"] = np.int64(len(sums))
    np.savez_compressed(os.path.join(HERE, "ops.npz"), **out)


def fit_case(R, rank, cfg):
    pair, traj = tropfact.fast_stmf(R, rank, cfg)
    st = strategies._SpecStrategy(strategies.FASTSTMF)
    g = np.random.default_rng(cfg.seed)
    work, ori = st.orient(R, g)
    U0, V0 = engine.random_acol_init(work, rank, cfg.acol_columns, g)
    return {
        "R": R.values, "M": R.mask, "rank": np.int64(rank), "seed": np.int64(cfg.seed),
        "sweeps": np.int64(cfg.budget_sweeps), "epsilon": np.float64(cfg.epsilon),
        "work_X": work.values, "work_M": work.mask, "transposed": np.bool_(ori.transposed),
        "perm": ori.row_perm.forward, "U0": U0, "V0": V0, "U": pair.U, "V": pair.V,
        "traj_t": np.array(traj.times), "traj_e": np.array(traj.errors),
    }


def c1_data(seed=0, mask_seed=1):
    """Config 1 (BASELINE.json configs[0]): 200x100 max-plus + N(0, 0.01), 20% hidden."""
    rng = np.random.default_rng(seed)
    A = rng.random((200, 3))
    B = rng.random((3, 100))
    X = tropical.trop_matmul(A, B) + rng.normal(0, 0.01, (200, 100))
    R, _ = datagen.apply_mask(X, 0.2, seed=mask_seed)
    return R


def make_fits():
    out = {}
    names = []
    rng = np.random.default_rng(7)
    small = [(12, 9, 2, 0.2, 6), (9, 15, 3, 0.3, 8), (25, 18, 3, 0.2, 5), (16, 40, 4, 0.5, 4),
             (30, 30, 1, 0.2, 5), (7, 5, 2, 0.0, 10)]
    for t, (m, n, r, frac, sweeps) in enumerate(small):
        A = rng.random((m, r))
        B = rng.random((r, n))
        X = tropical.trop_matmul(A, B) + rng.normal(0, 0.05, (m, n))
        R, _ = datagen.apply_mask(X, frac, seed=int(rng.integers(1 << 30)))
        cfg = engine.RunConfig(rank=r, budget_sweeps=sweeps, epsilon=0.0, seed=100 + t)
        names.append(f"s{t}")
        for k, v in fit_case(R, r, cfg).items():
            out[f"s{t}_{k}"] = v
    # convergence stop (default epsilon) on a small case
    R = c1_data(3, 4)
    R = tropical.MaskedMatrix(R.values[:40, :30], R.mask[:40, :30])
    cfg = engine.RunConfig(rank=3, budget_sweeps=50, epsilon=1e-8, seed=5)
    names.append("conv")
    for k, v in fit_case(R, 3, cfg).items():
        out[f"conv_{k}"] = v
    # config 1, first 3 sweeps (the full 100-sweep fit takes ~30 min in the reference)
    R = c1_data()
    cfg = engine.RunConfig(rank=3, budget_sweeps=3, epsilon=0.0, seed=42)
    names.append("c1")
    for k, v in fit_case(R, 3, cfg).items():
        out[f"c1_{k}"] = v
    out["names"] = np.array(names)
    np.savez_compressed(os.path.join(HERE, "fits.npz"), **out)


if __name__ == "__main__":
    make_ops()
    print("ops.npz written")
    make_fits()
    print("fits.npz written")
