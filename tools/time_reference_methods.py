"""Time the UNMODIFIED reference (tropfact, /root/reference/pkg/src) on every fit method
at config 1 (BASELINE.json configs[0]: 200x100 rank 3 fp64), wall-clock bounded.
Runs in the build container (the GPU box has no /root/reference); the output is
committed as profiles/r01_methods_reference_cpu.jsonl and read by bench_methods.py.

    python tools/time_reference_methods.py [seconds_per_method]
"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tropfact  # noqa: E402
from tropfact import engine  # noqa: E402

from paper_2205_06619_b200 import gen  # noqa: E402

METHODS = ["FastSTMF", "STMF", "STMF_ByElement_PermC_TD", "STMF_ByMatrix_NoPerm_TD_W",
           "STMF_ByRow_NoPerm_TD_W", "STMF_ByRow_PermR_TD_A_W", "STMF_ByRow_RandPermR_TD_B_W",
           "STMF_ByRow_RandPermR_SEQ_W"]


_count = {"attempts": 0, "sweeps": 0, "trials": 0}
_orig_attempt = engine.FitRun._attempt
_orig_mark = engine.FitRun.mark_sweep_boundary


def _attempt(self, *a):  # counts attempts without changing the reference's behaviour
    _count["attempts"] += 1
    return _orig_attempt(self, *a)


def _mark(self):
    _count["sweeps"] += 1
    return _orig_mark(self)


_orig_trial = engine.FitRun.trial


def _trial(self, *a):  # byrow_seq's trial evaluations (not attempts in the reference's count)
    _count["trials"] += 1
    return _orig_trial(self, *a)


engine.FitRun._attempt = _attempt
engine.FitRun.trial = _trial
engine.FitRun.mark_sweep_boundary = _mark


def main():
    secs = float(sys.argv[1]) if len(sys.argv) > 1 else 20.0
    R0 = gen.config1()
    R = tropfact.MaskedMatrix(np.where(R0.mask, R0.values, np.nan), R0.mask)
    out = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles",
                       "r01_methods_reference_cpu.jsonl")
    with open(out, "w") as f:
        for meth in METHODS:
            cfg = engine.RunConfig(rank=3, budget_seconds=secs, epsilon=0.0, seed=42)
            _count.update(attempts=0, sweeps=0, trials=0)
            t0 = time.perf_counter()
            pair, traj = tropfact.fit(R, 3, meth, cfg)
            wall = time.perf_counter() - t0
            rec = {"method": meth, "config": "config1 200x100 r3 fp64", "budget_s": secs, "wall_s": wall,
                   "attempts": _count["attempts"], "attempts_per_s": _count["attempts"] / wall,
                   "sweeps_completed": _count["sweeps"], "trials": _count["trials"],
                   "evaluations_per_s": (_count["attempts"] + _count["trials"]) / wall,
                   "samples": len(traj.errors), "err_init": traj.errors[0], "err_final": traj.errors[-1],
                   "cpu": "build container, 1 thread (numpy single-threaded)", "cores": 1}
            f.write(json.dumps(rec) + "\n")
            print(rec, flush=True)


if __name__ == "__main__":
    main()
