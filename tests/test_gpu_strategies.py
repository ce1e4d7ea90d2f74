"""Device parity of the reference's other fit methods: the STMF
baseline, ByElement, ByMatrix and every ByRow selection / permutation / shape, each
against the UNMODIFIED reference's fits (tests/golden/strategies.npz, written by
make_golden_strategies.py).  Bit-exact: factors and full trajectories."""

import numpy as np
import pytest

import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import _ext
from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def _golden():
    return np.load(f"{GOLDEN}/strategies.npz")


def _cases():
    g = _golden()
    return [str(x) for x in g["names"]]


@pytest.mark.parametrize("name", _cases())
def test_method_matches_reference(name):
    g = _golden()
    tag, meth = name.split("_", 1)
    R = pkg.MaskedMatrix(g[f"{tag}|R"], g[f"{tag}|M"])
    rank = int(g[f"{tag}|rank"])
    sweeps = int(g[f"{tag}|sweeps"]) * (4 if "ByMatrix" in meth else 1)
    cfg = pkg.RunConfig(rank=rank, budget_sweeps=sweeps, epsilon=0.0, seed=int(g["seed"]))
    pair, traj = pkg.fit(R, rank, meth, cfg)
    te = np.array(traj.errors)
    assert te.shape == g[f"{name}|traj_e"].shape, (te.size, g[f"{name}|traj_e"].size)
    assert np.array_equal(te, g[f"{name}|traj_e"])
    assert np.array_equal(np.array(traj.times), g[f"{name}|traj_t"])
    assert np.array_equal(pair.U, g[f"{name}|U"]) and np.array_equal(pair.V, g[f"{name}|V"])


def _np_td(X, M, U, V):
    P = np.max(U[:, :, None] + V[None, :, :], axis=1)  # trop_matmul (tropical.py:169)
    return np.where(M, np.abs(np.where(M, X, 0.0) - P), 0.0)  # td_grid (tropical.py:245)


def test_row_scores_and_matrix_candidates(ops):
    """td_grid(...).sum(axis=1) is numpy's pairwise row sum bit for bit; the ByMatrix
    candidate list is bymatrix_candidates' order (strategies.py:302-314)."""
    for c in range(int(ops["n_ops"])):
        X, M, U, V = (ops[f"c{c}_{k}"] for k in ("X", "M", "U", "V"))
        if not M.any(axis=0).all() or not M.any(axis=1).all():
            continue
        grid = _np_td(X, M, U, V)
        with _ext.Session(X, M, U.shape[1]) as s:
            s.set_factors(U, V)
            assert np.array_equal(s.row_scores(), grid.sum(axis=1)), c
            rows, cols, ks, sc = s.matrix_candidates()
        rs, cs = grid.sum(axis=1), grid.sum(axis=0)
        gi, gj = np.nonzero(M)
        scores = rs[gi] + cs[gj] - grid[gi, gj]
        order = np.argsort(-scores, kind="stable")
        arg = np.argmax(U[:, :, None] + V[None, :, :], axis=1)
        assert np.array_equal(rows, gi[order]) and np.array_equal(cols, gj[order]), c
        assert np.array_equal(ks, arg[gi[order], gj[order]]), c
        assert np.array_equal(sc, scores[order]), c


def test_row_scores_long_rows():
    """Rows longer than numpy's 128-element pairwise block (several tree levels)."""
    rng = np.random.default_rng(5)
    for m, n in ((3, 129), (5, 1000), (2, 4133)):
        X = rng.random((m, n)) * 4
        M = rng.random((m, n)) < 0.6
        M[:, 0] = True
        M[0, :] = True
        U = rng.random((m, 3))
        V = rng.random((3, n))
        with _ext.Session(X, M, 3) as s:
            s.set_factors(U, V)
            assert np.array_equal(s.row_scores(), _np_td(X, M, U, V).sum(axis=1)), (m, n)


def test_baseline_binary32_runs_exactly():
    """binary32 data: the baseline and ByElement run on the exact-sum objective."""
    from paper_2205_06619_b200 import gen
    R = gen.config3(m=48, n=64, rank=3)
    for meth in ("STMF", "STMF_ByElement_PermC_TD", "STMF_ByRow_NoPerm_TD_B", "STMF_ByRow_PermR_SEQ"):
        cfg = pkg.RunConfig(rank=3, budget_sweeps=2, epsilon=0.0, seed=3)
        pair, traj = pkg.fit(R, 3, meth, cfg)
        e = np.array(traj.errors)
        assert (np.diff(e) <= 0).all() and e[-1] < e[0], meth
        assert pkg.approx_error(R, pair.U, pair.V) == traj.final_error, meth
