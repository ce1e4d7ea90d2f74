"""A/B timing driver: sweep 2 of config C from the committed state S1 (bench.py's
step), REPS times, device time per sweep (CUDA events on the session stream).
Environment knobs select engine variants.

    python tools/s1_sweep.py [C] [REPS]
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("STMF_FIXPOINT_REPLAY", "0")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2205_06619_b200 import _ext  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
C, R, work, ori, U0, (U1, V1) = bench.workload(cfg)
N = int(work.mask.sum())
tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("STMF_") and k != "STMF_FIXPOINT_REPLAY")
with _ext.Session(work.values, work.mask, C["rank"]) as s:
    st = torch.cuda.ExternalStream(s.stream_handle())
    s.set_profiling(True)
    ms = []
    for r in range(reps + 1):
        s.set_factors(U1, V1)
        c0 = s.counters()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        tt, te, c = s.run(budget_sweeps=1, epsilon=0.0)
        e1.record(st)
        torch.cuda.synchronize()
        c1 = s.counters()
        if r:
            ms.append(e0.elapsed_time(e1))
    pb = (c1["phaseB_ns"] - c0["phaseB_ns"]) / 1e6
    print(f"[{tag or 'default'}] config {cfg} sweep 2: {min(ms):.1f} ms (all {[round(x) for x in ms]}), "
          f"attempts {c['attempts']} evaluated {c['evaluated']} err {te[-1]!r} "
          f"Gentries/s {c['attempts'] * N / min(ms) * 1e-6:.1f} phaseB {pb:.1f} ms "
          f"launches {c1['phaseB_timed'] - c0['phaseB_timed']}", flush=True)
