"""Edge shapes against the unmodified reference (tests/golden/edges.npz,
make_golden_edges.py): one row, one column, a fully given 2 x 2, rank above
min(m, n), quantised data full of exact ties, exact max-plus data fitted to ~1e-15 —
for FastSTMF and the other methods.  Factors and trajectories bit for bit."""

import numpy as np
import pytest

import paper_2205_06619_b200 as pkg
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _names():
    return [str(x) for x in np.load(f"{GOLDEN}/edges.npz")["names"]]


@pytest.mark.parametrize("name", _names())
def test_edge_case_matches_reference(name):
    g = np.load(f"{GOLDEN}/edges.npz")
    tag, meth = name.split("|")
    X, M, r = g[f"{tag}|X"], g[f"{tag}|M"], int(g[f"{tag}|rank"])
    R = pkg.MaskedMatrix(np.where(M, X, np.nan), M)
    cfg = pkg.RunConfig(rank=r, budget_sweeps=int(g[f"{name}|sweeps"]), epsilon=0.0, seed=7)
    pair, traj = pkg.fit(R, r, meth, cfg)
    assert np.array_equal(np.array(traj.errors), g[f"{name}|traj_e"])
    assert np.array_equal(np.array(traj.times), g[f"{name}|traj_t"])
    assert np.array_equal(pair.U, g[f"{name}|U"]) and np.array_equal(pair.V, g[f"{name}|V"])
