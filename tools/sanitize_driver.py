"""Small workload for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):
every kernel family of the library once, at toy sizes -- the sweep graph and the
host-driven loop in both precisions (fp64 replicas included), the attempt cap, the
other fit methods, the sharded engine (in-process group), the config-5 kernels
(dense TMA tiles and the sampled layout) and the metrics / b_norm entry points.

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2205_06619_b200 as pkg  # noqa: E402
from paper_2205_06619_b200 import _ext, engine, gen  # noqa: E402


def crop(R, m, n, dtype):
    return pkg.MaskedMatrix(R.values[:m, :n], R.mask[:m, :n], dtype=dtype)


def main():
    C1, C2 = gen.config1(), gen.config2()
    for dtype in (np.float64, np.float32):
        for graph in ("1", "0"):
            os.environ["STMF_GRAPH"] = graph
            R = crop(C2, 60, 90, dtype)
            p, t = pkg.fast_stmf(R, 5, pkg.RunConfig(rank=5, budget_sweeps=2, epsilon=0.0, seed=1))
            print(f"fit {np.dtype(dtype).name} graph={graph}: {len(t)} samples err {t.final_error:.6f}", flush=True)
    os.environ["STMF_GRAPH"] = "1"
    R = crop(C1, 50, 40, np.float64)
    work, _ = engine._orient_faststmf(R, np.random.default_rng(0))
    U0 = engine.acol_means(work, 3, 5, np.random.default_rng(1))
    with _ext.Session(work.values, work.mask, 3) as s:
        s.set_factors(U0)
        s.set_max_attempts(50)
        s.run(budget_sweeps=1, epsilon=0.0)
    for method in ("STMF", "STMF_ByRow_RandPermR_TD_W", "STMF_ByRow_RandPermR_TD_B_W", "STMF_ByRow_RandPermR_SEQ_W",
                   "STMF_ByElement_PermC_TD", "STMF_ByMatrix_NoPerm_TD"):
        pkg.fit(R, 3, method, pkg.RunConfig(rank=3, budget_sweeps=1, epsilon=0.0, seed=2))
        print("method", method, flush=True)
    Rf = crop(C2, 48, 70, np.float32)
    work, _ = engine._orient_faststmf(Rf, np.random.default_rng(0))
    U0 = engine.acol_means(work, 4, 5, np.random.default_rng(1))
    s = _ext.Session.sim_group(work.values, work.mask, 4, 3)
    s.set_factors(U0)
    s.run(budget_sweeps=1, epsilon=0.0)
    s.close()
    print("sharded sim group ok", flush=True)
    for layout in ("dense", "sampled"):
        r = _ext.bench_maxplus(256, 256, 8, 0.2, seed=3, reps=1, flush_l2=False, layout=layout)
        print("c5", layout, r["objective"], flush=True)
    a = np.random.default_rng(0).random(3000)
    print("b_norm", _ext.b_norm(a), flush=True)


if __name__ == "__main__":
    main()
