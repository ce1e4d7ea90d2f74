"""FastSTMF fit benchmark (BASELINE.json metric: observed-entry Gentries/s and fit
iters/sec), one JSON line on rank 0.

Workload (default): config 3 = BASELINE.json configs[2], the largest single-GPU
config: 4096 x 8192 max-plus + N(0, 0.05), 70% hidden, rank 10, binary32.  Seeded
synthetic data (paper_2205_06619_b200/gen.py; the paper's data is not available).

Window.  Every step is ONE ByRow/TD_A sweep (iteration) of the fit started from the
same committed state S1 -- the factors after sweep 1 of the seeded fit (fit seed 42,
tests/golden/c3_state_s1.npz, written by tools/make_states.py on the device and
re-derived bit for bit by this script's warm-up: `state_check`).  So every step is
sweep 2 of the fit, the same work each time, and the reference arm samples the same
sweep from the same state.

  value      Gentries/s = attempts x N_given / device time, attempts = candidate
             evaluations in reference order (FitRun._attempt calls, engine.py:278-295).
             Device time: CUDA events on the session stream around each sweep, L2
             flushed before each (the entry data, 340 MB, exceeds L2 anyway).
  e2e        the same metric through the public API from host arrays: each e2e step is
             one fast_stmf(R, 10, RunConfig(budget_sweeps=1), init=S1) call (H2D of X +
             mask + factors, orientation, caches, the sweep, D2H of U, V), wall-clock.
  --impl reference
             the UNMODIFIED reference (tropfact, numpy, installed into baseline/_ref)
             through its own stock code path: P = os.cpu_count() processes each build
             the reference's FitRun on the same work matrix and S1 factors (fp64: the
             reference's only precision) and run its ByRow/TD_A row visits
             (strategies.byrow_sweep, as _SpecStrategy.sweep calls it) on rows spread
             over the sweep, with the reference's own wall-clock budget; Gentries/s =
             sum of attempts x N / the longest process time.  No extrapolation.
  cpu_baseline  the same reference sample on 1 process (1 core).

N > 1 (torchrun): the row-sharded engine (distributed.py / stmf_shard.cuh: rows of X
and U split over the ranks, V replicated, NCCL collectives per row visit and batch);
total work fixed ("strong"), value = attempts x N / max-over-ranks device time.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]
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

METRIC = "FastSTMF fit observed-entry Gentries/s (attempts x given entries / s) and iters/sec (sweeps/s)"
PEAKS_PATH = os.path.join(ROOT, "MEASURED_PEAKS.json")
REF_PATH = os.path.join(ROOT, "baseline", "_ref")
FALLBACK_HBM = 6650.0
PHASEB_PROFILE = os.path.join(ROOT, "profiles", "r02_phaseB.json")


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--cpu-seconds", type=float, default=20.0, help="cpu_baseline sample (1 process)")
    ap.add_argument("--ref-seconds", type=float, default=None,
                    help="reference-arm sample per process (default: 6 s per step, 90..150 s)")
    ap.add_argument("--e2e-steps", type=int, default=3)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-c5", action="store_true", help="skip the config-5 kernel microbench")
    return ap.parse_args()


def state_path(cfg_no: int) -> str:
    return os.path.join(ROOT, "tests", "golden", f"c{cfg_no}_state_s1.npz")


def workload(cfg_no: int):
    """Config cfg_no, oriented and initialised exactly as fast_stmf does (seed 42)."""
    from paper_2205_06619_b200 import engine, gen
    C = gen.CONFIGS[cfg_no]
    R = C["make"]()
    rng = np.random.default_rng(42)
    work, ori = engine._orient_faststmf(R, rng)
    U0 = engine.acol_means(work, C["rank"], 5, rng)
    st = np.load(state_path(cfg_no))
    return C, R, work, ori, U0, (st["U"].astype(work.dtype), st["V"].astype(work.dtype))


def config_dict(cfg_no, C, work, n_gpus, extra=None):
    m, n = work.shape
    d = {"workload": f"config{cfg_no}: {m}x{n} work orientation, rank {C['rank']}, "
                     f"{C['dtype']}, {int(work.mask.sum())} given entries; "
                     f"1 step = 1 ByRow/TD_A sweep (sweep 2 of the seeded fit, from the committed state S1)",
         "rank": C["rank"], "m": m, "n": n, "given": int(work.mask.sum()),
         "parallelism": f"row-sharded x{n_gpus} (NCCL)" if n_gpus > 1 else "single",
         "window": "sweep 2 from S1 = tests/golden/c%d_state_s1.npz (state after sweep 1, fit seed 42)" % cfg_no,
         "l2": "flushed (256 MiB write) before every timed step; the entry data exceeds L2"}
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
# The reference's own code path (baseline/_ref: tropfact, unmodified numpy)
_REF = {}


def _ref_setup(cfg_no: int):
    """The reference's work matrix (its own orientation draws, seed 42) and the S1
    factors in binary64 (the reference computes in fp64 only, tropical.py:74)."""
    if REF_PATH not in sys.path:
        sys.path.insert(0, REF_PATH)
    import tropfact
    from tropfact import strategies as rs
    from paper_2205_06619_b200 import gen
    C = gen.CONFIGS[cfg_no]
    R = C["make"]()
    RR = tropfact.MaskedMatrix(np.where(R.mask, R.values.astype(np.float64), np.nan), R.mask)
    strat = rs._SpecStrategy(rs.FASTSTMF)
    work, _ = strat.orient(RR, np.random.default_rng(42))
    st = np.load(state_path(cfg_no))
    _REF.update(tropfact=tropfact, work=work, U=st["U"].astype(np.float64), V=st["V"].astype(np.float64),
                rank=C["rank"], N=int(work.mask.sum()))


def _ref_worker(args):
    """One process: the reference's FitRun on S1, then its row visits from row `start`
    on until its wall-clock budget (RunConfig.budget_seconds, checked by the
    reference between attempts, strategies.py:222) runs out."""
    start, seconds = args
    tf = _REF["tropfact"]
    from dataclasses import replace
    from tropfact import strategies as rs
    work = _REF["work"]
    cfg = tf.RunConfig(rank=_REF["rank"], budget_seconds=seconds, epsilon=0.0, seed=42)
    run = tf.engine.FitRun(work, _REF["U"].copy(), _REF["V"].copy(), cfg, wall_clock=True)
    run.current_sweep = 2
    # the budget counts from here (FitRun.__init__'s approx_error is setup, not sample)
    run.config = replace(cfg, budget_seconds=run.elapsed() + seconds)
    t0 = time.perf_counter()
    visits = 0
    for i in list(range(start, work.m)) + list(range(0, start)):
        if run.out_of_time():
            break
        rs.byrow_sweep(run, i, "TD_A")
        visits += 1
    dt = time.perf_counter() - t0
    return {"attempts": run.attempted_updates, "accepts": run.accepted_updates, "visits": visits, "seconds": dt}


def reference_sample(cfg_no: int, seconds: float, procs: int):
    """Aggregate Gentries/s of `procs` concurrent reference processes."""
    import multiprocessing as mp
    _ref_setup(cfg_no)
    m = _REF["work"].m
    starts = [(p * m) // procs for p in range(procs)]
    if procs == 1:
        res = [_ref_worker((starts[0], seconds))]
    else:
        with mp.get_context("fork").Pool(procs) as pool:
            res = pool.map(_ref_worker, [(s, seconds) for s in starts])
    att = sum(r["attempts"] for r in res)
    t = max(r["seconds"] for r in res)
    return {"gentries_per_s": att * _REF["N"] / t / 1e9, "attempts": att, "seconds": t,
            "visits": sum(r["visits"] for r in res), "accepts": sum(r["accepts"] for r in res), "procs": procs}


def ref_available() -> bool:
    return os.path.isdir(os.path.join(REF_PATH, "tropfact"))


def run_reference(args):
    """--impl reference: the unmodified reference on the host cores (rank 0 only)."""
    if int(os.environ.get("RANK", "0")) != 0:
        return
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "baseline/_ref/tropfact not installed (DESIGN.md)"}))
        return
    from paper_2205_06619_b200 import gen
    C = gen.CONFIGS[args.config]
    procs = os.cpu_count() or 1
    seconds = args.ref_seconds or float(min(150.0, max(90.0, 6.0 * args.steps)))
    if args.warmup > 0:  # untimed: page in numpy, the data and one row visit
        reference_sample(args.config, 2.0, 1)
    r = reference_sample(args.config, seconds, procs)
    work = _REF["work"]
    value = r["gentries_per_s"]
    sample = (f"{procs} processes (1 per host core, numpy single-threaded) of the unmodified reference "
              f"(baseline/_ref/tropfact): FitRun on the S1 state, then its byrow_sweep row visits from rows "
              f"spread over sweep 2, {seconds:.0f} s wall-clock budget each (RunConfig.budget_seconds); "
              f"{r['attempts']} attempts, {r['visits']} row visits, {r['accepts']} accepts")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "Gentries/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": r["seconds"] * 1e3 / max(args.steps, 1),
        "higher_is_better": True, "scaling": "strong" if args.gpus > 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (seeded, SURVEY.md §8d)",
        "config": config_dict(args.config, C, work, 1, {"reference_precision": "fp64 (tropical.py:74)"}),
        "attempts_per_s": r["attempts"] / r["seconds"],
        "cpu_baseline": {"value": value, "unit": "Gentries/s", "cores": procs, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": "Gentries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "consistency": {"timed_seconds": r["seconds"],
                        "note": "the steps are equal time slices of one sample; nothing is extrapolated"},
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
def phaseB_profile(cfg_no: int):
    try:
        return json.load(open(PHASEB_PROFILE)).get(str(cfg_no))
    except (OSError, ValueError):
        return None


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
    from paper_2205_06619_b200.distributed import ShardPlan, exchange_nccl_id
    _ext.lib()
    C, R, work, ori, U0, (U1, V1) = workload(args.config)
    m, n = work.shape
    N = int(work.mask.sum())
    r = C["rank"]
    if world > 1:
        if work.dtype != np.float32:
            raise SystemExit("the row-sharded engine is binary32: use --config 3 or 4 for N > 1")
        plan = ShardPlan(work, world, rank)
        s = _ext.Session.sharded(plan.rows(work.values), plan.rows(work.mask), r, m, plan.starts, plan.row_nnz,
                                 world, rank, exchange_nccl_id(dist), local)
        rows = plan.rows
        comm = s.comm_info()
    else:
        comm = None
        s = _ext.Session(work.values, work.mask, r, device=local)
        rows = lambda a: a  # noqa: E731
    stream = torch.cuda.ExternalStream(s.stream_handle(), device=torch.device("cuda", local))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # warm-up 1: sweep 1 from the seeded init must reproduce the committed S1 bit for bit
    s.set_factors(rows(U0))
    s.run(budget_sweeps=1, epsilon=0.0)
    Uc, Vc = s.get_factors()
    state_check = bool(np.array_equal(Uc, rows(U1)) and np.array_equal(Vc, V1))
    for _ in range(max(args.warmup - 1, 0)):
        s.set_factors(rows(U1), V1)
        s.run(budget_sweeps=1, epsilon=0.0)
    c0 = s.counters()
    times, attempts, accepts, evaluated, ends = [], [], [], [], []
    with ClockSampler(local) as clk:
        for _ in range(args.steps):
            s.set_factors(rows(U1), V1)  # every step is sweep 2 from S1 (untimed reset)
            flush.random_(0, 255)
            barrier()
            e0 = torch.cuda.Event(enable_timing=True)
            e1 = torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            tt, te, cnt = s.run(budget_sweeps=1, epsilon=0.0)
            e1.record(stream)
            barrier()
            times.append(e0.elapsed_time(e1) / 1e3)
            attempts.append(cnt["attempts"])
            accepts.append(cnt["accepts"])
            evaluated.append(cnt["evaluated"])
            ends.append(te[-1])
    c1 = s.counters()
    t_dev = sum(times)
    prof = None
    if world == 1:
        # phase-B launch times for the roofline: one more step, untimed, with CUDA
        # events around every phase-B launch (they perturb the step, so never timed)
        s.set_profiling(True)
        s.set_factors(rows(U1), V1)
        p0 = s.counters()
        _, _, pc = s.run(budget_sweeps=1, epsilon=0.0)
        prof = (p0, s.counters(), pc["evaluated"])
        s.set_profiling(False)
    if world > 1:
        t = torch.tensor([t_dev], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        t_dev = float(t[0])
    # attempts are global decisions (identical on every rank)
    value = sum(attempts) * N / t_dev / 1e9
    deterministic = len(set(attempts)) == 1 and len(set(ends)) == 1

    line = None
    if rank == 0:
        roof = roofline(args, work, prof, t_dev / args.steps, clk) if prof else None
        line = {
            "metric": METRIC, "value": value, "unit": "Gentries/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": t_dev * 1e3 / args.steps, "higher_is_better": True,
            "scaling": "strong" if world > 1 else "weak", "vs_baseline": None,
            "dtype": "f64" if work.dtype == np.float64 else "f32",
            "data": "synthetic (seeded generator of SURVEY.md §8d; no public dataset)",
            "config": config_dict(args.config, C, work, world),
            "sweeps_per_s": args.steps / t_dev,
            "attempts_per_step": attempts[0], "accepts_per_step": accepts[0], "evaluated_per_step": evaluated[0],
            "error_after_step": ends[0], "state_check": state_check, "deterministic_steps": deterministic,
            "gpu_launches": int(c1["launches"] - c0["launches"]),
            "comm": comm, "comm_nranks_ok": None if comm is None else (comm["nranks"] == world and comm["kind"] == "nccl"),
            "library_sorts": int(c1["cub_sorts"] - c0["cub_sorts"]),
            "roofline": roof,
            "clocks": clk.summary(),
        }
    s.close()
    del flush
    # e2e through the public API: fast_stmf from host arrays, warm-started at S1
    if not args.no_e2e:
        Uo, Vo = ori.restore(U1, V1)
        k_e2e = max(1, min(args.e2e_steps, args.steps))
        walls, e_att = [], []
        for _ in range(k_e2e):
            barrier()
            t0 = time.perf_counter()
            if world > 1:
                from paper_2205_06619_b200.distributed import fast_stmf_sharded
                pair, traj = fast_stmf_sharded(R, r, RunConfig(rank=r, budget_sweeps=1, epsilon=0.0, seed=42),
                                               device=local, init=(Uo, Vo))
            else:
                pair, traj = fast_stmf(R, r, RunConfig(rank=r, budget_sweeps=1, epsilon=0.0, seed=42),
                                       device=local, init=(Uo, Vo))
            torch.cuda.synchronize()
            dt = time.perf_counter() - t0
            if world > 1:
                t = torch.tensor([dt], dtype=torch.float64, device="cuda")
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                dt = float(t[0])
            walls.append(dt)
            e_att.append(traj.counts["attempts"])
        if rank == 0:
            h2d = R.m * R.n * (R.values.itemsize + 1) + (R.m + R.n) * r * R.values.itemsize
            d2h = (R.m + R.n) * r * R.values.itemsize + 16 * len(traj)
            line["e2e"] = {"value": sum(e_att) * N / sum(walls) / 1e9, "unit": "Gentries/s",
                           "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "steps": k_e2e,
                           "sweeps_per_s": k_e2e / sum(walls), "same_decisions": e_att[0] == attempts[0],
                           "note": "per step one fast_stmf(..., budget_sweeps=1, init=S1) call from host arrays "
                                   "(H2D X + mask + factors, orientation, caches, sweep 2, D2H U, V), wall clock"}
    # the kernel microbenchmark of BASELINE.json configs[4] at its largest HBM-bound point
    if rank == 0 and world == 1 and not args.no_c5:
        line["kernel_microbench"] = c5_microbench(_ext, local)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def roofline(args, work, prof, step_s, clk):
    """Phase B (k_phaseB: the candidate evaluations), the dominant kernel.

    achieved = algorithmic bytes of one launch / its average duration (CUDA events on
    the session stream around every launch, stmf_set_profiling).  One launch evaluates
    a whole speculative batch (E candidates x both rules) in one streaming of the given
    entries, so its algorithmic minimum is one attempt's data, 2 * B_pass with
    B_pass = N * s + ceil(m n / 8) (given values + bitmask).
    The resource phase B actually saturates is instruction issue (the per-(entry,
    evaluation) arithmetic), reported in `issue` from the committed ncu capture."""
    import torch
    m, n = work.shape
    N = int(work.mask.sum())
    s_bytes = work.dtype.itemsize
    b_pass = N * s_bytes + (m * n + 7) // 8
    c0, c1, evaluated = prof
    nb = c1["phaseB_timed"] - c0["phaseB_timed"]
    b_ns = c1["phaseB_ns"] - c0["phaseB_ns"]
    if not nb:
        return None
    avg_s = b_ns / 1e9 / nb
    peak, peak_src = peaks()
    achieved = 2 * b_pass / avg_s / 1e9
    prof = phaseB_profile(args.config) or {}
    rate = evaluated * N / (b_ns / 1e9)  # (entry, evaluation) pairs per second in phase B
    issue = l1 = None
    if "duration_us" in prof:
        # the binding resource: L1 data-pipe wavefronts (the gathers), scaled from the
        # capture's utilisation by the live (entry, evaluation) rate
        cap_rate = prof["evals"] * prof["given"] / (prof["duration_us"] * 1e-6)
        l1 = {"capture_frac": prof.get("l1_wavefront_frac"), "capture_pairs_per_s": cap_rate,
              "live_pairs_per_s": rate,
              "frac": prof.get("l1_wavefront_frac", 0) * rate / cap_rate if prof.get("l1_wavefront_frac") else None,
              "sectors_per_pair": prof.get("l1_global_ld_sectors", 0) / (prof["evals"] * prof["given"])}
    if "warp_instructions" in prof:
        ipe = prof["warp_instructions"] / (prof["evals"] * prof["given"])
        prop = torch.cuda.get_device_properties(0)
        sm_hz = (clk.summary().get("sm_mhz") or 1965.0) * 1e6
        ipeak = prop.multi_processor_count * 4 * sm_hz
        issue = {"warp_inst_per_entry_eval": ipe, "thread_inst_per_entry_eval": 32 * ipe,
                 "entry_evals_per_s": rate, "achieved_warp_inst_per_s": ipe * rate,
                 "peak_warp_inst_per_s": ipeak, "frac": ipe * rate / ipeak, "source": prof.get("capture")}
    traffic = prof.get("dram_bytes")
    return {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
            "traffic": traffic, "traffic_source": prof.get("capture"),
            # measured DRAM bytes per launch (launch list: one streaming of the entry data,
            # about the same for every batch size) over the live average launch time
            "dram_frac_measured": (traffic / avg_s / 1e9 / peak) if traffic else None,
            "kernel": "stmf::k_phaseB (candidate evaluation: 2nd residuation + error, both rules)",
            "algorithmic_bytes_per_launch": 2 * b_pass, "evals_per_launch": evaluated / nb,
            "avg_launch_us": avg_s * 1e6, "launches": nb, "share_of_step": (b_ns / 1e9) / step_s,
            "timing": "CUDA events around every phase-B launch of one extra (untimed) step",
            "peak_source": peak_src, "issue": issue, "l1": l1, "binding": "l1_wavefronts" if l1 else None,
            "note": "HBM is not phase B's bound: one launch serves a whole batch of evaluations from one "
                    "streaming of the entry data (traffic = that streaming incl. the product caches); the "
                    "binding resource is the L1 data pipe (the first-residuation gathers, roofline.l1), "
                    "instruction issue second (roofline.issue); profiles/r02_phaseB_c3.md"}


def c5_microbench(_ext, local):
    """BASELINE.json configs[4] at 65536^2, rank 4, density 1.0 (HBM-bound point)."""
    try:
        r5 = _ext.bench_maxplus(65536, 65536, 4, 1.0, seed=0, reps=5, flush_l2=True, device=local)
        peak, peak_src = peaks()
        out = {"config": "config5: m=n=65536, rank 4, density 1.0, fp32 (masked max-plus product + exact error)",
               "kernel": "stmf::k_maxplus_err (TMA-fed tiles)", "avg_ms": r5["avg_ms"],
               "roofline": {"bound": "hbm", "achieved": r5["gbs"], "peak": peak, "unit": "GB/s",
                            "frac": r5["gbs"] / peak, "traffic": 17753138000,
                            "traffic_source": "profiles/r01_c5_maxplus.md (ncu dram__bytes_read.sum)"},
               "objective": r5["objective"]}
        # the low-density point of the same config: only the given entries are stored, read and
        # computed (lane-coded records); achieved = the sampled layout's algorithmic bytes
        # m n / 8 + 4 given + factors over the launch time
        r1 = _ext.bench_maxplus(65536, 65536, 4, 0.1, seed=0, reps=5, flush_l2=True, device=local, layout="auto")
        out["low_density"] = {"config": "config5: m=n=65536, rank 4, density 0.1, fp32",
                              "kernel": "stmf::" + r1["kernel"], "avg_ms": r1["avg_ms"], "given": int(r1["given"]),
                              "roofline": {"bound": "hbm", "achieved": r1["gbs"], "peak": peak, "unit": "GB/s",
                                           "frac": r1["gbs"] / peak, "algorithmic_bytes": r1["bytes"]},
                              "objective": r1["objective"]}
        return out
    except Exception as e:  # noqa: BLE001 - reported, never fatal for the headline
        return {"error": str(e)}


def cpu_baseline(args):
    if not ref_available():
        return {"value": None, "unit": "Gentries/s", "cores": 0, "kind": "reference",
                "sample": "unavailable: baseline/_ref not installed"}
    r = reference_sample(args.config, args.cpu_seconds, 1)
    return {"value": r["gentries_per_s"], "unit": "Gentries/s", "cores": 1, "kind": "reference",
            "attempts_per_s": r["attempts"] / r["seconds"],
            "sample": f"the unmodified reference (baseline/_ref/tropfact, numpy, 1 process) on the S1 state: "
                      f"{r['attempts']} attempts in {r['visits']} row visits of sweep 2, {r['seconds']:.1f} s"}


def main():
    args = parse()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
