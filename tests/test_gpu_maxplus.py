"""Config-5 kernel (tiled masked max-plus product + exact error reduction) against
the CPU restatement on device-generated data; plus the dense prediction product."""

import math

import numpy as np
import pytest

import oracle
from paper_2205_06619_b200 import _ext

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,n,r,d", [(64, 128, 4, 1.0), (128, 256, 16, 0.5), (192, 128, 7, 0.1),
                                     (64, 384, 64, 0.3), (128, 128, 1, 0.9)])
def test_maxplus_err_matches_restatement(m, n, r, d):
    res = _ext.bench_maxplus(m, n, r, d, seed=m + n + r, reps=2, flush_l2=False, want_data=True)
    X, M, U, V = res["data"]
    assert res["given"] == M.sum()
    assert abs(M.mean() - d) < 0.1
    P, _, _ = oracle.trop_matmul(U, V)
    exact = math.fsum(np.abs(X[M] - P[M]).astype(np.float64).tolist())
    assert res["objective"] == exact
    assert res["objective"] == oracle.approx_error(np.where(M, X, np.nan).astype(np.float32), M, U, V)


def test_maxplus_rejects_unaligned():
    with pytest.raises(_ext.StmfError, match="multiple"):
        _ext.bench_maxplus(100, 128, 4, 0.5)
