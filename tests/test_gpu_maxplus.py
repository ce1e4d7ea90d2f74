"""Config-5 kernels (masked max-plus product + exact error reduction, BASELINE.json
configs[4]) against the CPU restatement on device-generated data: the dense-tile
kernel and the sampled (given-values-only) kernel, at toy shapes and at the config's
real 4096^2 (every rank x density) and 16384^2 (rank 4) points.  Both layouts compute
the exact sum of the binary32 residuals (tropical.py:214-222 restated in fp32), so
they agree with each other and with the restatement bit for bit."""

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


@pytest.mark.parametrize("m,n,r,d", [(128, 128, 4, 0.1), (256, 384, 13, 0.3), (384, 128, 64, 0.05),
                                     (128, 256, 1, 1.0), (256, 256, 33, 0.0)])
def test_sampled_layout_matches_dense_and_restatement(m, n, r, d):
    a = _ext.bench_maxplus(m, n, r, d, seed=7 * m + r, reps=1, flush_l2=False, layout="dense")
    b = _ext.bench_maxplus(m, n, r, d, seed=7 * m + r, reps=2, flush_l2=False, layout="sampled", want_data=True)
    assert b["layout"] == "sampled" and b["given"] == a["given"]
    assert b["objective"] == a["objective"]
    X, M, U, V = b["data"]
    assert b["objective"] == oracle.approx_error(np.where(M, X, np.nan).astype(np.float32), M, U, V)


@pytest.mark.parametrize("m,n,r,d", [(128, 2048, 4, 0.1), (256, 2048, 13, 0.3), (128, 1024, 16, 1.0),
                                     (384, 2048, 1, 0.5), (128, 1024, 8, 0.0), (640, 4096, 3, 0.02),
                                     (128, 768, 4, 0.2), (256, 2048, 4, 0.3)])
@pytest.mark.parametrize("stages,cpw", [(2, 8), (1, 1), (4, 2)])
def test_lane_compacted_kernel_matches_tiles_dense_and_restatement(m, n, r, d, stages, cpw, monkeypatch):
    """k_maxplus_err_lanes (lane-coded chunk records, bulk-copy stages) against the dense kernel,
    the tile kernel and the restatement; density 1.0 makes every record larger than a stage
    (read straight from global memory), 0.0 and 0.02 give empty chunks and lanes."""
    monkeypatch.setenv("STMF_C5_STAGES", str(stages))
    monkeypatch.setenv("STMF_C5_CPW", str(cpw))
    a = _ext.bench_maxplus(m, n, r, d, seed=3 * m + r, reps=1, flush_l2=False, layout="dense")
    t = _ext.bench_maxplus(m, n, r, d, seed=3 * m + r, reps=1, flush_l2=False, layout="tiles")
    b = _ext.bench_maxplus(m, n, r, d, seed=3 * m + r, reps=2, flush_l2=False, layout="lanes", want_data=True)
    assert b["kernel"] == "k_maxplus_err_lanes" and t["kernel"] == "k_maxplus_err_sampled"
    assert b["given"] == a["given"]
    assert b["objective"] == a["objective"] == t["objective"]
    X, M, U, V = b["data"]
    assert b["objective"] == oracle.approx_error(np.where(M, X, np.nan).astype(np.float32), M, U, V)


@pytest.mark.parametrize("span,r", [(s, r) for r in (4, 7) for s in (256, 512, 1024, 2048)
                                    if not (s == 2048 and r > 4)])
def test_lane_coded_kernel_every_chunk_width(span, r, monkeypatch):
    """The chunk width is chosen per matrix (the widest whose records fit a stage); every width
    gives the same exact objective (STMF_C5_SPAN forces one; 2048 exists at rank <= 4 only)."""
    a = _ext.bench_maxplus(256, 4096, r, 0.12, seed=41, reps=1, flush_l2=False, layout="dense")
    monkeypatch.setenv("STMF_C5_SPAN", str(span))
    b = _ext.bench_maxplus(256, 4096, r, 0.12, seed=41, reps=1, flush_l2=False, layout="lanes")
    assert b["kernel"] == "k_maxplus_err_lanes" and b["objective"] == a["objective"]


@pytest.mark.parametrize("r", [4, 16, 64])
@pytest.mark.parametrize("d", [0.1, 0.5, 1.0])
def test_config5_4096_matches_restatement(r, d):
    """BASELINE.json configs[4] at m = n = 4096: every (rank, density) point; the
    automatic layout choice, plus the other layout, against the restatement."""
    res = _ext.bench_maxplus(4096, 4096, r, d, seed=5, reps=1, flush_l2=False, want_data=True, layout="auto")
    X, M, U, V = res["data"]
    ref = oracle.approx_error(np.where(M, X, np.nan).astype(np.float32), M, U, V)
    assert res["objective"] == ref
    assert res["kernel"] == ("k_maxplus_err" if d > 0.35 else "k_maxplus_err_lanes" if r <= 16 else "k_maxplus_err_sampled")
    for other in ("dense", "tiles") + (("lanes",) if r <= 16 else ()):
        assert _ext.bench_maxplus(4096, 4096, r, d, seed=5, reps=1, flush_l2=False, layout=other)["objective"] == ref


def test_config5_16384_rank4_matches_restatement():
    res = _ext.bench_maxplus(16384, 16384, 4, 0.1, seed=9, reps=1, flush_l2=False, want_data=True, layout="auto")
    X, M, U, V = res["data"]
    assert res["layout"] == "sampled" and res["kernel"] == "k_maxplus_err_lanes"
    assert res["objective"] == oracle.approx_error(np.where(M, X, np.nan).astype(np.float32), M, U, V)


def test_maxplus_rejects_unaligned():
    with pytest.raises(_ext.StmfError, match="multiple"):
        _ext.bench_maxplus(100, 128, 4, 0.5)
    with pytest.raises(_ext.StmfError, match="multiples of 128"):
        _ext.bench_maxplus(64, 128, 4, 0.1, layout="sampled")
