"""Profiling driver: config C (default 3) from the committed state S1 (as bench.py's
timed step), one warm-up sweep, then sweep 2 inside cudaProfilerStart/Stop so that
`ncu --profile-from-start off` sees exactly one timed step.

    ncu --profile-from-start off --metrics gpu__time_duration.sum --csv python tools/phaseB_capture.py
    ncu --profile-from-start off --set full -k regex:k_phaseB -s 5 -c 1 python tools/phaseB_capture.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
os.environ.setdefault("STMF_FIXPOINT_REPLAY", "0")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2205_06619_b200 import _ext  # noqa: E402

cfg = int(sys.argv[1]) if len(sys.argv) > 1 else 3
C, R, work, ori, U0, (U1, V1) = bench.workload(cfg)
with _ext.Session(work.values, work.mask, C["rank"]) as s:
    s.set_factors(U1, V1)
    s.run(budget_sweeps=1, epsilon=0.0)
    s.set_factors(U1, V1)
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    tt, te, c = s.run(budget_sweeps=1, epsilon=0.0)
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    print(f"config {cfg}: sweep 2 attempts {c['attempts']} evaluated {c['evaluated']} err {te[-1]!r}")
