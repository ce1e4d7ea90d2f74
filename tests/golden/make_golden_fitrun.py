"""Golden fixture for the hand-driven protocol (tests/golden/fitrun.npz), generated from the
UNMODIFIED reference package (tropfact, read-only import from /root/reference/pkg/src).
Run in the build container:
    python tests/golden/make_golden_fitrun.py

One small seeded matrix, a Random-Acol start, then a fixed script of the reference's own
lower-level calls on one FitRun (engine.py:240-310, strategies.py:147-314): byrow_sweep with
every selection rule, byrow_seq, byelement_sweep, bymatrix_step, bymatrix_candidates, trial
and the select_k_* functions.  After every step the fixture records what the call returned,
the run's error and its attempt / accept counters; at the end the factors and the trajectory.
tests/test_gpu_fitrun.py replays the same script on the device-backed FitRun.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("STMF_REFERENCE", "/root/reference/pkg/src")
sys.path.insert(0, REF)
from tropfact import datagen, engine, strategies, tropical  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))

# the script: (function name, argument) — interpreted identically by the test
SCRIPT = ([("byrow", (i, "TD_A")) for i in range(0, 8)] + [("byrow", (i, "TD")) for i in range(8, 13)] +
          [("byrow", (i, "TD_B")) for i in range(13, 17)] + [("seq", 17), ("seq", 18), ("boundary", None),
                                                             ("byelement", None), ("boundary", None)] +
          [("bymatrix", None)] * 3 + [("byrow", (i, "SEQ")) for i in (19, 20)] + [("boundary", None)])


def main():
    rng = np.random.default_rng(5)
    m, n, r = 24, 30, 3
    A, B = rng.random((m, r)), rng.random((r, n))
    X = tropical.trop_matmul(A, B) + rng.normal(0, 0.05, (m, n))
    R, _ = datagen.apply_mask(X, 0.3, seed=77)
    U, V = engine.random_acol_init(R, r, 5, np.random.default_rng(9))
    out = {"values": np.where(R.mask, R.values, 0.0), "mask": R.mask, "U0": U.copy(), "V0": V.copy()}
    cfg = engine.RunConfig(rank=r, budget_sweeps=10, epsilon=0.0, seed=1)
    run = engine.FitRun(R, U, V, cfg, wall_clock=False)
    coin = np.random.default_rng(123)
    # pure selection functions and trials on the initial state
    probes = [(i, int(np.flatnonzero(R.mask[i])[i % 3])) for i in range(0, m, 3)]
    out["probes"] = np.array(probes)
    out["sel_td"] = np.array([strategies.select_k_td(U, V, i, j) for i, j in probes])
    out["sel_td_a"] = np.array([strategies.select_k_td_a(R, U, V, i, j) for i, j in probes])
    out["sel_td_b"] = np.array([strategies.select_k_td_b(R, U, V, i, j) for i, j in probes])
    out["trial_ulf"] = np.array([run.trial(engine.f_ulf, i, j, (i + j) % r) for i, j in probes])
    out["trial_urf"] = np.array([run.trial(engine.f_urf, i, j, (i + j) % r) for i, j in probes])
    cands = strategies.bymatrix_candidates(run)
    out["cand0"] = np.array([[c.i, c.j, c.k] for c in cands])
    out["cand0_score"] = np.array([c.err_score for c in cands])
    ret, errs, att, acc = [], [], [], []
    for name, arg in SCRIPT:
        if name == "byrow":
            res = strategies.byrow_sweep(run, arg[0], arg[1])
        elif name == "seq":
            res = strategies.byrow_seq(run, arg)
        elif name == "byelement":
            res = strategies.byelement_sweep(run)
        elif name == "bymatrix":
            res = strategies.bymatrix_step(run, coin)
        else:
            run.current_sweep += 1
            res = run.mark_sweep_boundary()
        ret.append(-1 if res is None else int(res))
        errs.append(run.err)
        att.append(run.attempted_updates)
        acc.append(run.accepted_updates)
        print(name, arg, res, run.err, run.attempted_updates, run.accepted_updates, flush=True)
    cands = strategies.bymatrix_candidates(run)
    out["cand1"] = np.array([[c.i, c.j, c.k] for c in cands])
    out["cand1_score"] = np.array([c.err_score for c in cands])
    out.update(ret=np.array(ret), err=np.array(errs), attempted=np.array(att), accepted=np.array(acc),
               U=run.U, V=run.V, traj_t=np.array(run.trajectory.times), traj_e=np.array(run.trajectory.errors))
    np.savez_compressed(os.path.join(HERE, "fitrun.npz"), **out)
    print("wrote fitrun.npz:", len(SCRIPT), "steps,", run.attempted_updates, "attempts")


if __name__ == "__main__":
    main()
