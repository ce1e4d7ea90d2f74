"""Bounded fit throughput for the large configs (C3, C4) and the small ones (C1)
on one B200, plus the in-process sharded engine on the same work.  One JSON line
per run:  sweeps or row visits completed in a wall-clock budget, attempts/s,
observed-entry Gentries/s (attempts * N / t), evaluated (speculative) evals.

  python bench_fit.py --config 4 --seconds 30 [--shards 1,4]
"""

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
# benchmarks execute every sweep: no replay of fixpoint sweeps (stmf_replayed_sweeps)
os.environ["STMF_FIXPOINT_REPLAY"] = "0"
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--seconds", type=float, default=20.0)
    ap.add_argument("--sweeps", type=int, default=0, help="sweep budget instead of seconds")
    ap.add_argument("--shards", default="0", help="0 = single-GPU engine; G>0 = in-process sharded engine")
    ap.add_argument("--warm-sweeps", type=int, default=0)
    args = ap.parse_args()
    from paper_2205_06619_b200 import _ext, engine, gen
    C = gen.CONFIGS[args.config]
    t = time.perf_counter()
    R = C["make"]()
    t_gen = time.perf_counter() - t
    rng = np.random.default_rng(42)
    work, _ = engine._orient_faststmf(R, rng)
    U0 = engine.acol_means(work, C["rank"], 5, rng)
    N = int(work.mask.sum())
    for g in (int(x) for x in args.shards.split(",")):
        t = time.perf_counter()
        if g == 0:
            s = _ext.Session(work.values, work.mask, C["rank"])
        else:
            s = _ext.Session.sim_group(work.values, work.mask, C["rank"], g)
        s.set_factors(U0)
        t_setup = time.perf_counter() - t
        for _ in range(args.warm_sweeps):
            s.run(budget_sweeps=1, epsilon=0.0)
        t = time.perf_counter()
        if args.sweeps:
            tt, te, c = s.run(budget_sweeps=args.sweeps, epsilon=0.0)
        else:
            tt, te, c = s.run(budget_seconds=args.seconds, epsilon=0.0)
        dt = time.perf_counter() - t
        s.close()
        line = {"config": args.config, "engine": "single" if g == 0 else f"sim_sharded_{g}",
                "m": work.m, "n": work.n, "rank": C["rank"], "given": N,
                "dtype": str(work.dtype), "gen_s": t_gen, "setup_s": t_setup, "run_s": dt,
                "warm_sweeps": args.warm_sweeps, "sweeps_done": c["sweeps"], "row_visits": c["row_visits"],
                "attempts": c["attempts"], "accepts": c["accepts"], "evaluated": c["evaluated"],
                "attempts_per_s": c["attempts"] / dt, "row_visits_per_s": c["row_visits"] / dt,
                "gentries_per_s": c["attempts"] * N / dt / 1e9,
                "err_first": float(te[0]), "err_last": float(te[-1]), "traj_len": int(len(te))}
        print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
