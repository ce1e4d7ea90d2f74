"""Binary32 parity at the real config shapes (BASELINE.json configs[2] and [3]):
the device engine replays the first K attempts of sweep 1 that the C restatement
made (tests/golden/make_golden_fp32_shapes.py, oracle.fit(max_attempts=K)) and must
reproduce its trajectory, counts and factors bit for bit.  The restatement follows
engine.py:313-348 / strategies.py:191-224 with the exact-sum objective
(tropical.py:214-222 restated in binary32).

The capped runs use the host-driven sweep loop (stmf_set_max_attempts); the config-3
case also runs its full first sweep through the per-sweep CUDA graph and checks the
graph's accept sequence against the same prefix."""

import os
import sys

import numpy as np
import pytest

from paper_2205_06619_b200 import _ext

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden"))
from make_golden_fp32_shapes import OUT, STATES, late_V, prepare, sha  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def fx():
    return np.load(OUT)


def _check_inputs(fx, name, work, U0):
    X, M = work.values, work.mask
    assert tuple(fx[f"{name}_shape"]) == work.shape
    assert str(fx[f"{name}_sha_M"]) == sha(M), "generator drift (mask)"
    assert str(fx[f"{name}_sha_X"]) == sha(np.where(M, X, 0)), "generator drift (values)"
    assert str(fx[f"{name}_sha_U0"]) == sha(U0), "init drift"


@pytest.mark.parametrize("name", ["c4s", "c3", "c3late", "c3fix", pytest.param("c4", marks=pytest.mark.slow)])
def test_capped_sweep1_prefix_matches_restatement(fx, name):
    """c3late starts from the device's state after 24 sweeps of config 3 (stored in the
    fixtures): the restatement's next K attempts, reproduced bit for bit.  c3fix starts from
    the state after sweep 41, the fit's fixpoint: the restatement and the device both reject
    every candidate of the first row visit."""
    work, U0, rank, K = prepare(name)
    assert int(fx[f"{name}_K"]) == K
    _check_inputs(fx, name, work, U0)
    with _ext.Session(work.values, work.mask, rank) as s:
        # V0 = (-U0)^T (x)* R on the device (engine.py:194), or the stored late state's V
        s.set_factors(U0, late_V(work, name) if name in STATES else None)
        assert sha(s.get_factors()[1]) == str(fx[f"{name}_sha_V0"])
        s.set_max_attempts(K)
        tt, te, cnt = s.run(budget_sweeps=1, epsilon=0.0)
        U, V = s.get_factors()
    assert cnt["attempts"] == int(fx[f"{name}_attempts"])
    assert cnt["accepts"] == int(fx[f"{name}_accepts"])
    if name == "c3fix":
        assert cnt["accepts"] == 0 and cnt["attempts"] == K and te[0] == te[-1] == 1353413.1359968781
    assert np.array_equal(te, fx[f"{name}_traj_e"])
    assert np.array_equal(tt, fx[f"{name}_traj_t"])
    assert np.array_equal(U[:64], fx[f"{name}_U_head"])
    assert np.array_equal(V[:, :256], fx[f"{name}_V_head"])
    assert sha(U) == str(fx[f"{name}_sha_U"]) and sha(V) == str(fx[f"{name}_sha_V"])


def test_config3_graph_sweep_prefix_matches_restatement(fx):
    """The full first sweep through the sweep graph: its accept sequence starts with
    the restatement's K-attempt prefix (every sample but the cap's final boundary)."""
    name = "c3"
    work, U0, rank, K = prepare(name)
    ref = fx[f"{name}_traj_e"]
    with _ext.Session(work.values, work.mask, rank) as s:
        s.set_factors(U0)
        tt, te, cnt = s.run(budget_sweeps=1, epsilon=0.0)
    assert cnt["sweeps"] == 1 and len(te) > len(ref)
    assert np.array_equal(te[:len(ref) - 1], ref[:-1])
    # the objective never increases and the boundary repeats the last accept
    assert np.all(np.diff(te) <= 0) and te[-1] == te[-2]
