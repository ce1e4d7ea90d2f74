"""Every reference fit method on one B200 at config 1
(BASELINE.json configs[0]: 200x100 rank 3 fp64), through the public API
(``fit(R, rank, method, RunConfig)``: host orientation + init, device sweeps, D2H).
One JSON line per method: sweeps, attempts, wall time, attempts/s, Gentries/s
(attempts * N / t), and the reference's attempts/s on the same workload from
profiles/r01_methods_reference_cpu.jsonl (tools/time_reference_methods.py, 1 CPU
thread in the build container; /root/reference is not on the GPU box).

  python bench_methods.py [--sweeps 10]
"""

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
# benchmarks execute every sweep: no replay of fixpoint sweeps (stmf_replayed_sweeps)
os.environ["STMF_FIXPOINT_REPLAY"] = "0"
sys.path.insert(0, ROOT)

METHODS = ["FastSTMF", "STMF", "STMF_ByElement_PermC_TD", "STMF_ByMatrix_NoPerm_TD_W",
           "STMF_ByRow_NoPerm_TD_W", "STMF_ByRow_PermR_TD_A_W", "STMF_ByRow_RandPermR_TD_B_W",
           "STMF_ByRow_RandPermR_SEQ_W"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweeps", type=int, default=10)
    args = ap.parse_args()
    import paper_2205_06619_b200 as pkg
    from paper_2205_06619_b200 import gen
    ref = {}
    p = os.path.join(ROOT, "profiles", "r01_methods_reference_cpu.jsonl")
    if os.path.exists(p):
        for line in open(p):
            r = json.loads(line)
            ref[r["method"]] = r
    R = gen.config1()
    N = R.given_count
    # warm the library / context once
    pkg.fast_stmf(R, 3, pkg.RunConfig(rank=3, budget_sweeps=1, epsilon=0.0, seed=1))
    for meth in METHODS:
        sweeps = args.sweeps
        cfg = pkg.RunConfig(rank=3, budget_sweeps=sweeps, epsilon=0.0, seed=42)
        t = time.perf_counter()
        pair, traj = pkg.fit(R, 3, meth, cfg)
        wall = time.perf_counter() - t
        c = traj.counts
        rec = {"method": meth, "config": "config1 200x100 r3 fp64", "sweeps": c["sweeps"], "wall_s": wall,
               "attempts": c["attempts"], "accepts": c["accepts"], "evaluated": c["evaluated"],
               "attempts_per_s": c["attempts"] / wall, "sweeps_per_s": c["sweeps"] / wall,
               "gentries_per_s": c["attempts"] * N / wall / 1e9, "final_error": traj.final_error,
               "timing": "wall clock of one fit() call: host orientation + Acol draws, H2D, device sweeps, D2H"}
        if meth in ref:
            r = ref[meth]
            # the comparable unit: attempts (FitRun._attempt calls) for most methods;
            # trial evaluations for SEQ (byrow_seq trials every (j, k, rule)); whole
            # steps for ByMatrix (one accepted update per sweep)
            if "SEQ" in meth:
                unit, gpu, cpu = "evaluations/s", c["evaluated"] / wall, r["evaluations_per_s"]
            elif "ByMatrix" in meth:
                unit, gpu, cpu = "sweeps/s", rec["sweeps_per_s"], r["sweeps_completed"] / r["wall_s"]
            else:
                unit, gpu, cpu = "attempts/s", rec["attempts_per_s"], r["attempts_per_s"]
            rec["reference_cpu"] = {"value": cpu, "unit": unit, "cores": r["cores"],
                                    "sample": f"{r['budget_s']:.0f} s wall-clock budget of the reference fit, "
                                              f"{r['cpu']}"}
            rec["speedup_vs_reference"] = {"unit": unit, "gpu": gpu, "ratio": gpu / cpu}
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
