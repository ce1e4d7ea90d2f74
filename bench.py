"""FastSTMF fit benchmark (BASELINE.json metric: fit iters/sec = sweeps/s, plus
observed-entry Gentries/s), one JSON line on rank 0.

Default workload: config 2 (BASELINE.json configs[1]: 500x1000 log2(1+lognormal),
50% hidden, rank 5, fp64) — one step = one full ByRow/TD_A sweep of the fit with
the factors resident in HBM.  W warm-up sweeps from the seeded Random-Acol init,
then K timed sweeps (CUDA events on the session stream, L2 flushed before each
step; the working set is L2-sized, so the flush only removes cross-step reuse).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

N > 1 (torchrun): config 2 does not shard (too small), so each rank
runs an independent replica fit (seed 42 + rank) — "replicas only"; value = total
sweeps of all ranks / max-over-ranks device time.

--impl reference: the CPU restatement of the reference (oracle/, the reference is
pure numpy and cannot be compiled) on the host cores: one independent fit per
thread, each a bounded sample of sweep 1 from the same seeded init;
sweeps/s = attempts/s / (attempts in sweep 1).  A sweep's attempt count is a
property of the fit trajectory, identical on every implementation that makes the
reference's decisions (tests/test_gpu_parity.py); SWEEP1_ATTEMPTS holds it.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
# benchmarks execute every sweep: no replay of fixpoint sweeps (stmf_replayed_sweeps)
os.environ["STMF_FIXPOINT_REPLAY"] = "0"
sys.path.insert(0, ROOT)

METRIC = "FastSTMF fit iters/sec (sweeps/s) and observed-entry Gentries/s"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
# attempts (reference-order candidate evaluations) in sweep 1 from the seeded init
# (fit seed 42): config 1 from the oracle, configs 2-3 from the device engine
# (bit-identical decisions, tests/test_gpu_parity.py)
SWEEP1_ATTEMPTS = {1: 1383, 2: 83025, 3: 226759}
FALLBACK_HBM = 6650.0


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU baseline sample budget")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the config-5 kernel microbench")
    return ap.parse_args()


def workload(cfg_no: int, rank_id: int = 0):
    from paper_2205_06619_b200 import engine, gen
    C = gen.CONFIGS[cfg_no]
    R = C["make"]()
    rng = np.random.default_rng(42 + rank_id)
    work, ori = engine._orient_faststmf(R, rng)
    U0 = engine.acol_means(work, C["rank"], 5, rng)
    return C, R, work, U0


def config_dict(cfg_no, C, work, n_gpus, extra=None):
    m, n = work.shape
    d = {"workload": f"config{cfg_no}: {m}x{n} work orientation, rank {C['rank']}, "
                     f"{'fp64' if work.dtype == np.float64 else 'fp32'}, "
                     f"{int(work.mask.sum())} given entries; 1 step = 1 ByRow/TD_A sweep",
         "rank": C["rank"], "m": m, "n": n, "given": int(work.mask.sum()),
         "parallelism": "replicas" if n_gpus > 1 else "single",
         "l2": "flushed (256 MiB write) before every timed step; working set is L2-sized"}
    if extra:
        d.update(extra)
    return d


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm = [float(r[0]) for r in self.rows if len(r) >= 7 and r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if len(r) >= 7 and r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) >= 7 for i in range(4) if r[3 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


def peaks():
    try:
        with open(PEAKS_PATH) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return FALLBACK_HBM, "fallback (B200_PROFILING.md)"


# ----------------------------------------------------------------------------
def cpu_sample(work, U0, V0, seconds: float, threads: int = 1):
    """The oracle port on `threads` independent copies of the same fit, bounded to
    ~`seconds` of CPU work each; returns (row visits/s, attempts/s) aggregated."""
    import oracle
    oracle.build()
    X, M = work.values, work.mask
    # calibrate: attempts per second of one fit
    t = time.perf_counter()
    probe = oracle.fit(X, M, U0, V0, budget_sweeps=1, epsilon=0.0, max_attempts=20)
    per_attempt = max((time.perf_counter() - t) / max(probe["attempts"], 1), 1e-6)
    cap = max(40, int(seconds / per_attempt))
    results = [None] * threads

    def one(ti):
        t0 = time.perf_counter()
        r = oracle.fit(X, M, U0, V0, budget_sweeps=1, epsilon=0.0, max_attempts=cap)
        results[ti] = (r, time.perf_counter() - t0)

    ths = [threading.Thread(target=one, args=(i,)) for i in range(threads)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    visits = sum(r["row_visits"] for r, _ in results)
    attempts = sum(r["attempts"] for r, _ in results)
    wall = max(dt for _, dt in results)
    return visits / wall, attempts / wall, cap, results[0][0]


def run_reference(args):
    """--impl reference: the CPU port of the reference's fit on the host cores."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from paper_2205_06619_b200 import gen
    C, R, work, U0 = workload(args.config)
    import oracle
    V0 = np.stack([oracle.residuate_row(work.values, work.mask, U0[:, k]) for k in range(C["rank"])])
    threads = os.cpu_count() or 1
    m = work.shape[0]
    N = int(work.mask.sum())
    vals = []
    gent = []
    for _ in range(args.warmup):
        cpu_sample(work, U0, V0, min(2.0, args.cpu_seconds / 4), 1)
    for _ in range(args.steps):
        vps, aps, cap, r0 = cpu_sample(work, U0, V0, args.cpu_seconds / max(args.steps, 1), threads)
        vals.append(aps / SWEEP1_ATTEMPTS[args.config])
        gent.append(aps * N / 1e9)
    value = float(np.mean(vals))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 / value if value else None,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64" if work.dtype == np.float64 else "f32", "data": "synthetic (seeded, SURVEY.md §8d)",
        "config": config_dict(args.config, C, work, 1),
        "gentries_per_s": float(np.mean(gent)),
        "cpu_baseline": {"value": value, "unit": "sweeps/s", "cores": threads, "kind": "port",
                         "sample": f"{threads} independent fits (1 per host thread) of sweep 1 from the seeded "
                                   f"init, each capped at {cap} attempts; sweeps/s = aggregate attempts/s / "
                                   f"{SWEEP1_ATTEMPTS[args.config]} attempts per sweep 1 "
                                   f"(the reference is numpy-only; oracle/ is its C restatement)"},
        "e2e": {"value": value, "unit": "sweeps/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
def run_b200(args):
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    torch.cuda.set_device(local)
    from paper_2205_06619_b200 import _ext, fast_stmf, RunConfig
    _ext.lib()
    C, R, work, U0 = workload(args.config, rank)
    m, n = work.shape
    N = int(work.mask.sum())
    s = _ext.Session(work.values, work.mask, C["rank"], device=local)
    s.set_factors(U0)
    V0 = s.get_factors()[1]
    s.set_profiling(True)
    stream = torch.cuda.ExternalStream(s.stream_handle(), device=torch.device("cuda", local))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for _ in range(args.warmup):
        s.run(budget_sweeps=1, epsilon=0.0)
    U_w, V_w = s.get_factors()
    c0 = s.counters()
    total_ms = 0.0
    attempts = accepts = evaluated = 0
    first_step_attempts = None
    traj_end = None
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            flush.random_(0, 255)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tt, te, cnt = s.run(budget_sweeps=1, epsilon=0.0)
            e1.record(stream)
            barrier()
            total_ms += e0.elapsed_time(e1)
            attempts += cnt["attempts"]
            if first_step_attempts is None:
                first_step_attempts = cnt["attempts"]
            accepts += cnt["accepts"]
            evaluated += cnt["evaluated"]
            traj_end = te[-1]
    c1 = s.counters()
    t_dev = total_ms / 1e3
    if world > 1:
        t = torch.tensor([t_dev, attempts], dtype=torch.float64, device="cuda")
        tmax = t.clone()
        dist.all_reduce(tmax[:1], op=dist.ReduceOp.MAX)
        dist.all_reduce(t[1:], op=dist.ReduceOp.SUM)
        t_dev_max, attempts_all = float(tmax[0]), float(t[1])
    else:
        t_dev_max, attempts_all = t_dev, float(attempts)
    value = args.steps * world / t_dev_max
    gentries = attempts_all * N / t_dev_max / 1e9

    # roofline of the dominant kernel (phase B).  SURVEY.md §8(d): one attempt (a
    # candidate evaluation over all N given entries) needs B_attempt = 2 * B_pass
    # algorithmic bytes, B_pass = N*s + ceil(m*n/8) (values + bitmask); one launch
    # evaluates every candidate of its batch (both rules), so its algorithmic bytes
    # are B_attempt * (evaluations in the launch).  Launch times: CUDA events on the
    # session stream around every phase-B launch (stmf_set_profiling).
    s_bytes = work.dtype.itemsize
    b_pass = N * s_bytes + (m * n + 7) // 8
    nb = c1["phaseB_timed"] - c0["phaseB_timed"]
    b_ns = c1["phaseB_ns"] - c0["phaseB_ns"]
    avg_s = b_ns / 1e9 / max(nb, 1)
    evals_per_launch = evaluated / max(nb, 1)
    b_launch = 2 * b_pass * evals_per_launch
    peak, peak_src = peaks()
    achieved = b_launch / avg_s / 1e9 if nb else None
    l2_resident = 2 * N * (3 * s_bytes + 5) < 0.5 * 126e6
    traffic, traffic_src = None, None
    try:
        tr = json.load(open(os.path.join(ROOT, "profiles", "r01_phaseB_traffic.json"))).get(str(args.config))
        if tr:
            traffic, traffic_src = tr["bytes"], tr["capture"]
    except (OSError, ValueError):
        pass
    # the binding resource is instruction issue (profiles/r01_v4_phaseB.md): warp
    # instructions per (entry, evaluation) from the committed ncu capture, times the
    # live (entry, evaluation) rate, against the issue peak of the SMs
    issue = None
    try:
        ti = json.load(open(os.path.join(ROOT, "profiles", "r01_phaseB_traffic.json"))).get(str(args.config), {})
        ti = ti.get("issue")
        if ti and nb:
            ipe = ti["warp_instructions"] / (ti["evals"] * ti["given"])
            rate = evals_per_launch * N / avg_s
            prop = torch.cuda.get_device_properties(local)
            sm_hz = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
            ipeak = prop.multi_processor_count * 4 * sm_hz
            issue = {"warp_inst_per_entry_eval": ipe, "entry_evals_per_s": rate,
                     "achieved_warp_inst_per_s": ipe * rate, "peak_warp_inst_per_s": ipeak,
                     "frac": ipe * rate / ipeak, "source": ti["capture"]}
    except (OSError, ValueError, KeyError):
        pass
    roofline = {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak if achieved else None, "traffic": traffic, "traffic_source": traffic_src,
                "kernel": "stmf::k_phaseB (candidate evaluation: 2nd residuation + error, both rules)",
                "bytes_per_launch": b_launch, "bytes_per_attempt": 2 * b_pass,
                "evals_per_launch": evals_per_launch, "avg_launch_us": avg_s * 1e6, "launches": nb,
                "share_of_step": (b_ns / 1e9) / t_dev if t_dev else None, "peak_source": peak_src,
                "issue": issue,
                "note": ("one pass over the given entries serves a group of 8 evaluations and the working "
                         "set is L2-resident, so the HBM-equivalent rate can exceed the HBM peak; the binding "
                         "resource is instruction issue (roofline.issue; DESIGN.md, profiles/r01_v4_phaseB.md)")
                        if l2_resident else
                        "one pass over the given entries serves a group of 8 evaluations (DESIGN.md)"}

    line = None
    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "sweeps/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev_max * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None,
            "dtype": "f64" if work.dtype == np.float64 else "f32",
            "data": "synthetic (seeded generator of SURVEY.md §8d; no public dataset)",
            "config": config_dict(args.config, C, work, world),
            "gentries_per_s": gentries,
            "attempts_per_step": attempts / args.steps, "accepts_per_step": accepts / args.steps,
            "evaluated_per_step": evaluated / args.steps, "final_error": traj_end,
            "gpu_launches": int(c1["launches"] - c0["launches"]),
            "library_sorts": int(c1["cub_sorts"] - c0["cub_sorts"]),
            "roofline": roofline,
            "clocks": clk.summary(),
        }
    # e2e through the public API: host MaskedMatrix -> fast_stmf (H2D of X + mask,
    # init, K sweeps from the seeded init, D2H of U, V) timed on the host
    # the timed session's device memory returns to the library's pool, which the e2e
    # fit below then reuses (as a second fit in a user's process would)
    s.close()
    del flush
    if not args.no_e2e:
        barrier()
        t0 = time.perf_counter()
        cfg = RunConfig(rank=C["rank"], budget_sweeps=args.steps, epsilon=0.0, seed=42 + rank)
        pair, traj = fast_stmf(R, C["rank"], cfg, device=local)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
        if world > 1:
            t = torch.tensor([dt], dtype=torch.float64, device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            dt = float(t[0])
        if rank == 0:
            h2d = R.m * R.n * (R.values.itemsize + 1) + R.m * C["rank"] * R.values.itemsize
            d2h = (R.m + R.n) * C["rank"] * R.values.itemsize + 16 * len(traj)
            line["e2e"] = {"value": args.steps * world / dt, "unit": "sweeps/s",
                           "h2d_bytes_per_step": h2d // args.steps, "d2h_bytes_per_step": d2h // args.steps,
                           "note": "one fast_stmf call per run: H2D, init, K sweeps from init, D2H"}
    # the kernel microbenchmark of BASELINE.json configs[4] at its largest HBM-bound point
    # (masked max-plus product + exact error, 65536^2, rank 4, density 1.0; device-generated
    # data, L2 flushed between reps), so the bench line carries that kernel's roofline too
    if rank == 0 and not args.no_c5:
        try:
            r5 = _ext.bench_maxplus(65536, 65536, 4, 1.0, seed=0, reps=5, flush_l2=True, device=local)
            peak, peak_src = peaks()
            line["kernel_microbench"] = {
                "config": "config5: m=n=65536, rank 4, density 1.0, fp32 (masked max-plus product + exact error)",
                "kernel": "stmf::k_maxplus_err (TMA-fed tiles)", "avg_ms": r5["avg_ms"],
                "roofline": {"bound": "hbm", "achieved": r5["gbs"], "peak": peak, "unit": "GB/s",
                             "frac": r5["gbs"] / peak, "traffic": 17753138000,
                             "traffic_source": "profiles/r01_c5_maxplus.md (ncu dram__bytes_read.sum)"},
                "objective": r5["objective"]}
        except Exception as e:  # noqa: BLE001 - reported, never fatal for the headline
            line["kernel_microbench"] = {"error": str(e)}
    if rank == 0 and not args.no_cpu_baseline:
        vps, aps, cap, r0 = cpu_sample(work, U_w, V_w, args.cpu_seconds, 1)
        cps = aps / first_step_attempts
        line["cpu_baseline"] = {
            "value": cps, "unit": "sweeps/s", "cores": 1, "kind": "port",
            "attempts_per_s": aps, "gentries_per_s": aps * N / 1e9,
            "sample": f"oracle/ C restatement, 1 thread, from the same post-warm-up factors: the first "
                      f"{r0['attempts']} attempts of sweep {args.warmup + 1}; sweeps/s = attempts/s / "
                      f"{first_step_attempts} (that sweep's attempt count, identical decisions)"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
