"""Host logic of the row-sharded path on CPU: the row partition, and a world-size-2
gloo run of fast_stmf_sharded (NCCL-id exchange, per-rank shard rows, U
assembly, orientation restore).  The device session is replaced by the CPU
restatement (oracle/, the checker) so this runs without a GPU."""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import distributed as D
from paper_2205_06619_b200 import engine


def test_row_blocks_balanced_and_contiguous():
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 4, 8):
        nnz = rng.integers(1, 100, size=257)
        s = D.row_blocks(nnz, world)
        assert s[0] == 0 and s[-1] == 257 and np.all(np.diff(s) >= 1)
        per = np.add.reduceat(nnz, s[:-1])
        assert per.max() - per.min() <= 2 * nnz.max() + 1
    with pytest.raises(ValueError):
        D.row_blocks(np.ones(3), 4)


class OracleShard:
    """CPU stand-in for one shard: runs the restatement on the whole work matrix
    (every rank computes the same fit) and exposes this rank's rows of U."""

    def __init__(self, plan, work, rank):
        self.plan, self.work, self.rank = plan, work, rank

    def set_factors(self, U_rows, V=None):
        # the full U0 is rebuilt from every rank's rows by the caller's all-gather
        # at the end; here each rank needs it whole: gather it now
        parts = [None] * dist.get_world_size()
        dist.all_gather_object(parts, np.asarray(U_rows))
        self.U0 = np.concatenate(parts)
        self.V0 = np.stack([oracle.residuate_row(self.work.values, self.work.mask, self.U0[:, k])
                            for k in range(self.rank)])

    def run(self, budget_sweeps, budget_seconds, epsilon):
        self.res = oracle.fit(self.work.values, self.work.mask, self.U0, self.V0,
                              budget_sweeps=budget_sweeps, epsilon=epsilon)
        return self.res["traj_t"], self.res["traj_err"], {"attempts": self.res["attempts"]}

    def get_factors(self):
        return self.plan.rows(self.res["U"]), self.res["V"]


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        rng = np.random.default_rng(3)
        m, n, r = 20, 14, 2  # tall: exercises the transpose in orient/restore
        A = rng.random((m, r)); B = rng.random((r, n))
        X = (np.max(A[:, :, None] + B[None], axis=1) + rng.normal(0, 0.05, (m, n))).astype(np.float32)
        M = rng.random((m, n)) > 0.25
        M[:, 0] = True; M[0, :] = True
        R = pkg.MaskedMatrix(X, M, dtype=np.float32)
        cfg = pkg.RunConfig(rank=r, budget_sweeps=3, epsilon=0.0, seed=9)
        ids = []

        def factory(plan, work, rank_, nccl_id):
            ids.append(nccl_id)
            assert plan.world == world and plan.rank == rank
            return OracleShard(plan, work, rank_)

        # the id exchange needs the library only on rank 0 (GPU-free here)
        D.exchange_nccl_id = lambda d=None: b"test-id" if world > 1 else None
        pair, traj = D.fast_stmf_sharded(R, r, cfg, session_factory=factory)
        out[rank] = (pair.U, pair.V, np.array(traj.errors), ids[0])
    finally:
        dist.destroy_process_group()


def test_gloo_world2_sharded_driver_matches_single_process():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    # reference: the same fit in one process
    rng = np.random.default_rng(3)
    m, n, r = 20, 14, 2
    A = rng.random((m, r)); B = rng.random((r, n))
    X = (np.max(A[:, :, None] + B[None], axis=1) + rng.normal(0, 0.05, (m, n))).astype(np.float32)
    M = rng.random((m, n)) > 0.25
    M[:, 0] = True; M[0, :] = True
    R = pkg.MaskedMatrix(X, M, dtype=np.float32)
    g = np.random.default_rng(9)
    work, ori = engine._orient_faststmf(R, g)
    U0 = engine.acol_means(work, r, 5, g)
    V0 = np.stack([oracle.residuate_row(work.values, work.mask, U0[:, k]) for k in range(r)])
    ref = oracle.fit(work.values, work.mask, U0, V0, budget_sweeps=3, epsilon=0.0)
    U, V = ori.restore(ref["U"], ref["V"])
    for rank in range(world):
        Ur, Vr, er, nid = out[rank]
        assert nid == b"test-id"
        assert np.array_equal(Ur, U) and np.array_equal(Vr, V)
        assert np.array_equal(er, ref["traj_err"])
