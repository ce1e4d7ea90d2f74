"""Golden values of the reference's host-side statistics and sidecar files
(tests/golden/hoststats.npz + hoststats_files/), from the UNMODIFIED reference
(metrics.py, io.py).  python tests/golden/make_golden_hoststats.py"""
import os
import shutil
import sys

import numpy as np

sys.path.insert(0, os.environ.get("STMF_REFERENCE", "/root/reference/pkg/src"))
from tropfact import engine, io, metrics, tropical  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(17)


def traj(t_max, n, e0):
    tr = engine.Trajectory(t_init=0.0, t_max=t_max, time_unit="sweeps")
    t = np.sort(rng.random(n) * t_max)
    e = e0 * np.cumprod(1 - 0.1 * rng.random(n))
    for a, b in zip(t, e):
        tr.append(float(a), float(b))
    return tr


base = traj(10.0, 12, 100.0)
other = traj(10.0, 9, 120.0)
grid = metrics.make_grid(10.0, 0.7)
out = {
    "base_t": np.array(base.times), "base_e": np.array(base.errors),
    "other_t": np.array(other.times), "other_e": np.array(other.errors),
    "grid": grid, "grid2": metrics.make_grid(3.0, 1.0, 0.5),
    "ne": metrics.normalized_error(other, base, grid),
    "interp": metrics.step_interpolate(base.times, base.errors, grid),
}
samples = rng.random(40)
out["samples"] = samples
out["ci"] = np.array(metrics.bootstrap_ci(samples, n_resamples=300, level=0.9, seed=3))
scores = rng.random((4, 6))
scores[1, 2] = scores[0, 2]
scores[3, 4] = np.inf
scores[2, 4] = np.inf
out["scores"] = scores
out["ranks"] = metrics.rank_methods(scores)
out["ranks_hi"] = metrics.rank_methods(scores, lower_is_better=False)
out["avg"] = metrics.average_ranks(out["ranks"])
out["cd"] = np.array([metrics.nemenyi_cd(4, 6), metrics.nemenyi_cd(3, 10, 0.1)])
out["ttr"] = np.array([metrics.time_to_reach(base, float(base.errors[5]), grid),
                       metrics.time_to_reach(base, -1.0, grid)])
out["omega"] = np.array(metrics.omega(samples[:20], samples[20:]))
np.savez_compressed(os.path.join(HERE, "hoststats.npz"), **out)

files = os.path.join(HERE, "hoststats_files")
shutil.rmtree(files, ignore_errors=True)
os.makedirs(files)
io.save_trajectory(os.path.join(files, "traj.jsonl"), base)
U = rng.random((5, 2))
V = rng.random((2, 4))
ori = engine.Orientation(True, tropical.Permutation(np.array([1, 0])), None)
io.save_factors(files, engine.FactorPair(U, V, 2, ori), config={"seed": 3, "method": "FastSTMF"}, prefix="p_")
X = rng.random((4, 5))
train, test = __import__("tropfact").datagen.apply_mask(X, 0.3, seed=2)
io.save_dataset(os.path.join(files, "ds"), train, test, X, {"name": "toy", "lam": 0.5}, A=U[:4], B=V)
print("hoststats written")
