"""Audit mode (RunConfig.audit, engine.py:143-153, 279-294) and the attempt-cap test
hook (stmf_set_max_attempts, the checker's oracle.fit(max_attempts=...)) on the
device, against the CPU restatement."""

import numpy as np
import pytest

import oracle
import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import _ext, engine, gen

pytestmark = pytest.mark.gpu


def _work(R, rank, seed=42):
    rng = np.random.default_rng(seed)
    work, _ = engine._orient_faststmf(R, rng)
    U0 = engine.acol_means(work, rank, 5, rng)
    return work, U0


def _crop(R, m, n, dtype=None):
    return pkg.MaskedMatrix(R.values[:m, :n], R.mask[:m, :n], dtype=dtype or R.dtype)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_audit_fit_equals_plain_fit(dtype):
    R = _crop(gen.config1(), 120, 80, dtype)
    base = dict(rank=3, budget_sweeps=3, epsilon=0.0, seed=7)
    p0, t0 = pkg.fast_stmf(R, 3, pkg.RunConfig(**base))
    p1, t1 = pkg.fast_stmf(R, 3, pkg.RunConfig(**base, audit=True))
    assert np.array_equal(p0.U, p1.U) and np.array_equal(p0.V, p1.V)
    assert np.array_equal(np.array(t0.errors), np.array(t1.errors))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("K", [1, 2, 7, 40, 333, 1000])
def test_attempt_cap_matches_restatement(dtype, K):
    R = _crop(gen.config2(), 90, 160, dtype)
    work, U0 = _work(R, 5)
    U0 = U0.astype(dtype)
    V0 = np.stack([oracle.residuate_row(work.values, work.mask, U0[:, k]) for k in range(5)])
    ref = oracle.fit(work.values, work.mask, U0, V0, budget_sweeps=3, epsilon=0.0, max_attempts=K)
    with _ext.Session(work.values, work.mask, 5) as s:
        s.set_factors(U0, V0)
        s.set_max_attempts(K)
        tt, te, cnt = s.run(budget_sweeps=3, epsilon=0.0)
        U, V = s.get_factors()
    assert ref["capped"] and cnt["attempts"] == ref["attempts"] == K
    assert cnt["accepts"] == ref["accepts"]
    assert np.array_equal(te, ref["traj_err"]) and np.array_equal(tt, ref["traj_t"])
    assert np.array_equal(U, ref["U"]) and np.array_equal(V, ref["V"])


def test_attempt_cap_rejects_seq_selection():
    R = _crop(gen.config1(), 40, 30)
    work, U0 = _work(R, 3)
    with _ext.Session(work.values, work.mask, 3) as s:
        s.set_factors(U0)
        s.set_strategy(_ext.FAMILY_BYROW, _ext.SEL_SEQ)
        s.set_max_attempts(5)
        with pytest.raises(_ext.StmfError, match="attempt cap"):
            s.run(budget_sweeps=1, epsilon=0.0)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_warm_start_continues_the_fit(dtype):
    """fast_stmf(init=...) from the factors after sweep 1 reaches the 2-sweep fit's
    factors bit for bit (ByRow sweeps draw no random numbers)."""
    R = _crop(gen.config2(), 150, 90, dtype)  # tall: exercises the transposed orientation
    p1, _ = pkg.fast_stmf(R, 5, pkg.RunConfig(rank=5, budget_sweeps=1, epsilon=0.0, seed=3))
    p2, t2 = pkg.fast_stmf(R, 5, pkg.RunConfig(rank=5, budget_sweeps=2, epsilon=0.0, seed=3))
    pw, tw = pkg.fast_stmf(R, 5, pkg.RunConfig(rank=5, budget_sweeps=1, epsilon=0.0, seed=3), init=(p1.U, p1.V))
    assert np.array_equal(pw.U, p2.U) and np.array_equal(pw.V, p2.V)
    assert tw.errors[0] == t2.errors[len(t2.errors) - len(tw.errors)]
    assert tw.errors[-1] == t2.errors[-1]
