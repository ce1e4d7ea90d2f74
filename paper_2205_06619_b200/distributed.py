"""Row-sharded FastSTMF across the GPUs of one box.

One process per GPU (torchrun).  Every rank holds the host matrix, runs the same
host orientation + Random-Acol draws (identical by seed), and creates its shard:
a contiguous block of work rows with about N/world given entries.  The fit runs in
the CUDA library with NCCL collectives between the ranks (stmf_create_sharded);
``torch.distributed`` only carries the NCCL unique id and gathers U at the end.
All reductions are exact, so results are bit-identical for any world size and
equal to the single-GPU binary32 fit.
"""

from __future__ import annotations

import time

import numpy as np

from . import _ext
from .engine import _orient_faststmf, acol_means
from .types import FactorPair, MaskedMatrix, RunConfig, Trajectory

__all__ = ["row_blocks", "fast_stmf_sharded", "ShardPlan"]


def row_blocks(row_nnz, world: int) -> np.ndarray:
    """Contiguous row blocks [starts[s], starts[s+1]) with ~equal given counts
    (same rule as the library's in-process groups); every block is non-empty."""
    nnz = np.asarray(row_nnz, dtype=np.int64)
    m = nnz.size
    if world < 1 or world > m:
        raise ValueError(f"cannot split {m} rows over {world} shards")
    N = int(nnz.sum())
    starts = np.zeros(world + 1, np.int64)
    starts[world] = m
    acc = 0
    r = 0
    for s in range(1, world):
        target = N * s // world
        while r < m - (world - s) and acc + nnz[r] <= target:
            acc += int(nnz[r])
            r += 1
        r = max(r, int(starts[s - 1]) + 1)
        starts[s] = r
    return starts


class ShardPlan:
    """This rank's part of a sharded fit."""

    def __init__(self, work: MaskedMatrix, world: int, rank: int):
        self.row_nnz = work.mask.sum(axis=1).astype(np.int64)
        self.starts = row_blocks(self.row_nnz, world)
        self.world, self.rank = world, rank
        self.r0, self.r1 = int(self.starts[rank]), int(self.starts[rank + 1])

    def rows(self, a):
        return a[self.r0:self.r1]


def _dist():
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        raise RuntimeError("fast_stmf_sharded needs an initialised torch.distributed process group")
    return dist


def exchange_nccl_id(dist=None) -> bytes | None:
    """NCCL unique id created on rank 0 and broadcast to every rank."""
    dist = dist or _dist()
    if dist.get_world_size() == 1:
        return None
    obj = [None]
    if dist.get_rank() == 0:
        buf = (np.zeros(256, np.uint8))
        size = np.array([256], np.int64)
        import ctypes
        _ext._check(_ext.lib().stmf_nccl_unique_id(_ext._p(buf), size.ctypes.data_as(ctypes.POINTER(ctypes.c_int64))))
        obj[0] = bytes(buf[: int(size[0])])
    dist.broadcast_object_list(obj, src=0)
    return obj[0]


def fast_stmf_sharded(R: MaskedMatrix, rank: int, config: RunConfig, device: int | None = None,
                      session_factory=None, init=None):
    """fast_stmf with the work rows sharded over the ranks of the default process
    group (binary32).  Returns (FactorPair, Trajectory) on every rank.

    ``session_factory(plan, work, rank, nccl_id)`` may replace the device session
    (host-logic tests on CPU); it must return an object with set_factors / run /
    get_factors like ``_ext.Session``.  ``init``: optional warm-start (U, V) in the
    original orientation (engine.run_fit).
    """
    dist = _dist()
    world, me = dist.get_world_size(), dist.get_rank()
    if R.dtype != np.float32:
        R = MaskedMatrix(R.values, R.mask, dtype=np.float32)
    config.validate()
    R.validate_coverage()
    rng = np.random.default_rng(config.seed)
    wall = config.budget_seconds is not None
    t0 = time.perf_counter()
    work, orientation = _orient_faststmf(R, rng)
    V0 = None
    if init is None:
        U0 = acol_means(work, rank, config.acol_columns, rng)
    else:
        U0, V0 = orientation.apply_factors(np.asarray(init[0], np.float32), np.asarray(init[1], np.float32))
    plan = ShardPlan(work, world, me)
    nccl_id = exchange_nccl_id(dist)
    if session_factory is None:
        s = _ext.Session.sharded(plan.rows(work.values), plan.rows(work.mask), rank, work.m, plan.starts,
                                 plan.row_nnz, world, me, nccl_id, device)
    else:
        s = session_factory(plan, work, rank, nccl_id)
    s.set_factors(plan.rows(U0), V0)
    t_init = time.perf_counter() - t0 if wall else 0.0
    budget_seconds = max(config.budget_seconds - t_init, 1e-9) if wall else None
    tt, te, counts = s.run(config.budget_sweeps, budget_seconds, config.epsilon)
    U_loc, V = s.get_factors()
    if hasattr(s, "close"):
        s.close()
    parts = [None] * world
    dist.all_gather_object(parts, U_loc)
    U = np.concatenate(parts, axis=0)
    traj = Trajectory(t_init=t_init, t_max=config.budget_seconds if wall else float(config.budget_sweeps),
                      time_unit="seconds" if wall else "sweeps")
    for t, e in zip(tt.tolist(), te.tolist()):
        traj.append(t + (t_init if wall else 0.0), e)
    traj.counts = counts
    U_out, V_out = orientation.restore(U, V)
    return FactorPair(U_out, V_out, rank, orientation), traj
