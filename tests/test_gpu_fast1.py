"""Phase B's first half from per-line order statistics (stmf_fast1.cuh) against the
full passes over the given entries: identical trajectories, counts and factors in
both precisions, through the sweep graph and the host-driven loop, on shapes where
the statistics walk falls back (short lines, non-uniform factor indices) and where
it does not.  (Every other GPU test runs with the statistics path, the default.)"""

import os

import numpy as np
import pytest

import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import _ext, engine, gen

pytestmark = pytest.mark.gpu


def _fit(work, U0, rank, sweeps, fast1, graph):
    old = {k: os.environ.get(k) for k in ("STMF_FAST1", "STMF_GRAPH")}
    os.environ["STMF_FAST1"] = "1" if fast1 else "0"
    os.environ["STMF_GRAPH"] = "1" if graph else "0"
    try:
        with _ext.Session(work.values, work.mask, rank) as s:
            s.set_factors(U0)
            tt, te, c = s.run(budget_sweeps=sweeps, epsilon=0.0)
            U, V = s.get_factors()
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v
    return te, U, V, c


@pytest.mark.parametrize("cfg,m,n,rank,dtype,sweeps", [
    (2, 200, 400, 5, np.float64, 3),
    (2, 120, 300, 5, np.float32, 3),
    (3, 256, 512, 10, np.float32, 2),
    (1, 100, 100, 3, np.float64, 4),
])
@pytest.mark.parametrize("graph", [True, False])
def test_statistics_walk_equals_full_pass(cfg, m, n, rank, dtype, sweeps, graph):
    R = gen.CONFIGS[cfg]["make"]()
    R = pkg.MaskedMatrix(R.values[:m, :n], R.mask[:m, :n], dtype=dtype)
    rng = np.random.default_rng(42)
    work, _ = engine._orient_faststmf(R, rng)
    U0 = engine.acol_means(work, rank, 5, rng)
    a = _fit(work, U0, rank, sweeps, False, graph)
    b = _fit(work, U0, rank, sweeps, True, graph)
    assert np.array_equal(a[0], b[0])
    assert np.array_equal(a[1], b[1]) and np.array_equal(a[2], b[2])
    assert a[3]["attempts"] == b[3]["attempts"] and a[3]["accepts"] == b[3]["accepts"]
