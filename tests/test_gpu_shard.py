"""Shard invariance on one B200: the row-sharded engine with 1..4 in-process
shards (collectives as kernels over the shards' buffers) gives bit-identical
trajectories, factors and attempt counts to the single-GPU engine and to the CPU
restatement."""

import numpy as np
import pytest

import oracle
import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import _ext, engine

pytestmark = pytest.mark.gpu


def _case(seed, m, n, r, frac):
    rng = np.random.default_rng(seed)
    A = rng.random((m, r)); B = rng.random((r, n))
    X = (np.max(A[:, :, None] + B[None], axis=1) + rng.normal(0, 0.05, (m, n))).astype(np.float32)
    M = rng.random((m, n)) >= frac
    M[np.arange(m), rng.integers(0, n, m)] = True
    M[rng.integers(0, m, n), np.arange(n)] = True
    R = pkg.MaskedMatrix(X, M, dtype=np.float32)
    work, _ = engine._orient_faststmf(R, np.random.default_rng(seed + 1))
    U0 = engine.acol_means(work, r, 5, np.random.default_rng(seed + 2))
    return work, U0


def _single(work, U0, r, sweeps):
    with _ext.Session(work.values, work.mask, r) as s:
        s.set_factors(U0)
        scores = s.col_scores()  # of the initial state
        tt, te, c = s.run(budget_sweeps=sweeps, epsilon=0.0)
        U, V = s.get_factors()
    return te, U, V, c, scores


@pytest.mark.parametrize("seed,m,n,r,frac,sweeps", [(11, 40, 70, 3, 0.3, 3), (12, 96, 150, 6, 0.7, 2),
                                                     (13, 64, 64, 10, 0.5, 2)])
def test_sim_groups_match_single_engine(seed, m, n, r, frac, sweeps):
    work, U0 = _case(seed, m, n, r, frac)
    te1, U1, V1, c1, sc1 = _single(work, U0, r, sweeps)
    for shards in (1, 2, 3, 4):
        s = _ext.Session.sim_group(work.values, work.mask, r, shards)
        try:
            s.set_factors(U0)
            assert np.array_equal(s.col_scores(), sc1), shards
            tt, te, c = s.run(budget_sweeps=sweeps, epsilon=0.0)
            U, V = s.get_factors()
        finally:
            s.close()
        assert np.array_equal(te, te1), shards
        assert np.array_equal(U, U1) and np.array_equal(V, V1), shards
        assert c["attempts"] == c1["attempts"] and c["accepts"] == c1["accepts"], shards


def test_sim_group_matches_restatement():
    work, U0 = _case(21, 48, 90, 4, 0.6)
    V0 = np.stack([oracle.residuate_row(work.values, work.mask, U0[:, k]) for k in range(4)])
    ref = oracle.fit(work.values, work.mask, U0, V0, budget_sweeps=2, epsilon=0.0)
    s = _ext.Session.sim_group(work.values, work.mask, 4, 3)
    try:
        s.set_factors(U0)
        tt, te, c = s.run(budget_sweeps=2, epsilon=0.0)
        U, V = s.get_factors()
    finally:
        s.close()
    assert np.array_equal(te, ref["traj_err"])
    assert np.array_equal(U, ref["U"]) and np.array_equal(V, ref["V"])


def test_sharded_world1_is_the_nccl_entry_point():
    work, U0 = _case(31, 30, 45, 3, 0.4)
    nnz = work.mask.sum(axis=1)
    s = _ext.Session.sharded(work.values, work.mask, 3, work.m, np.array([0, work.m]), nnz, 1, 0, None)
    try:
        s.set_factors(U0)
        tt, te, c = s.run(budget_sweeps=2, epsilon=0.0)
    finally:
        s.close()
    te1, *_ = _single(work, U0, 3, 2)
    assert np.array_equal(te, te1)


def _nccl_id():
    import ctypes
    buf = np.zeros(256, np.uint8)
    size = np.array([256], np.int64)
    _ext._check(_ext.lib().stmf_nccl_unique_id(_ext._p(buf), size.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
    return bytes(buf[: int(size[0])])


@pytest.mark.parametrize("seed,m,n,r,frac,sweeps", [(41, 60, 90, 4, 0.5, 3), (42, 128, 200, 10, 0.7, 2)])
def test_sharded_world1_over_a_real_nccl_communicator(seed, m, n, r, frac, sweeps):
    """stmf_create_sharded with an NCCL id at world size 1: ncclCommInitRank(nranks=1)
    and every collective of the sharded engine (MIN on binary32, SUM on int64 limbs,
    all-gather, broadcast) execute through libnccl, and the fit equals the
    single-device engine bit for bit."""
    work, U0 = _case(seed, m, n, r, frac)
    te1, U1, V1, c1, _ = _single(work, U0, r, sweeps)
    nnz = work.mask.sum(axis=1)
    s = _ext.Session.sharded(work.values, work.mask, r, work.m, np.array([0, work.m]), nnz, 1, 0, _nccl_id())
    try:
        assert s.comm_info() == {"nranks": 1, "rank": 0, "kind": "nccl"}
        s.set_factors(U0)
        tt, te, c = s.run(budget_sweeps=sweeps, epsilon=0.0)
        U, V = s.get_factors()
    finally:
        s.close()
    assert np.array_equal(te, te1)
    assert np.array_equal(U, U1) and np.array_equal(V, V1)
    assert c["attempts"] == c1["attempts"]


def test_sharded_rejects_fp64():
    X = np.ones((4, 5))
    M = np.ones((4, 5), bool)
    with pytest.raises(_ext.StmfError, match="binary32"):
        _ext.lib()
        import ctypes
        h = ctypes.c_void_p()
        _ext._check(_ext.lib().stmf_create_sim_group(ctypes.byref(h), _ext.STMF_F64, 4, 5, 1, _ext._p(X),
                                                     _ext._p(M.astype(np.uint8)), 2, 0))
