"""The CPU restatement (oracle/) pinned against the reference's own outputs
(tests/golden/*.npz, made by tests/golden/make_golden.py from the unmodified
reference) and the SPEC's worked examples.  CPU only."""

import math

import numpy as np
import pytest

import oracle
from conftest import fit_case


def test_ops_match_reference(ops):
    for c in range(int(ops["n_ops"])):
        g = lambda k: ops[f"c{c}_{k}"]  # noqa: E731
        X, M, U, V = g("X"), g("M"), g("U"), g("V")
        P, arg, top2 = oracle.trop_matmul(U, V)
        assert np.array_equal(P, g("P")), c
        assert np.array_equal(arg, g("arg")), c
        assert np.array_equal(oracle.col_scores(X, M, U, V), g("scores")), c
        assert np.array_equal(oracle.residuate_row(X, M, g("u")), g("rr")), c
        assert np.array_equal(oracle.residuate_col(X, M, g("v")), g("rc")), c
        assert oracle.approx_error(X, M, U, V) == float(g("err")), c
        i, j, k = (int(x) for x in g("ijk"))
        U1, V1, f1 = oracle.f_ulf(X, M, U, V, i, j, k)
        assert np.array_equal(U1, g("ulf_U")) and np.array_equal(V1, g("ulf_V")) and f1 == float(g("ulf_f")), c
        U2, V2, f2 = oracle.f_urf(X, M, U, V, i, j, k)
        assert np.array_equal(U2, g("urf_U")) and np.array_equal(V2, g("urf_V")) and f2 == float(g("urf_f")), c


def test_top2_is_second_best(ops):
    U, V = ops["c3_U"], ops["c3_V"]
    P, arg, top2 = oracle.trop_matmul(U, V)
    S = U[:, :, None] + V[None, :, :]
    m, r, n = S.shape
    for i in range(m):
        for j in range(n):
            others = [S[i, l, j] for l in range(r) if l != arg[i, j]]
            assert top2[i, j] == (max(others) if others else -np.inf)


def test_b_norm_numpy_pairwise(ops):
    sums = ops["bn_sums"]
    for t in range(int(ops["n_bn"])):
        assert oracle.b_norm(ops[f"bn{t}_w"]) == sums[t], t


def test_b_norm_f32_is_exact_sum():
    rng = np.random.default_rng(3)
    for n in (0, 1, 7, 8, 129, 5000, 100_000):
        w = (rng.normal(size=n) * rng.random(n) ** 20).astype(np.float32)
        w[: n // 10] = 0
        exact = math.fsum(np.abs(w.astype(np.float64)).tolist())
        assert oracle.b_norm(w) == exact
    # subnormals and huge values
    w = np.array([1e-45, 3e-44, 1e38, 2.5, -7e-40], np.float32)
    assert oracle.b_norm(w) == math.fsum(np.abs(w.astype(np.float64)).tolist())


@pytest.mark.parametrize("name", ["s0", "s1", "s2", "s3", "s4", "s5", "conv", "c1"])
def test_fit_matches_reference(fits, name):
    c = fit_case(fits, name)
    res = oracle.fit(c["work_X"], c["work_M"], c["U0"], c["V0"], budget_sweeps=int(c["sweeps"]),
                     epsilon=float(c["epsilon"]))
    assert np.array_equal(res["traj_err"], c["traj_e"])
    assert np.array_equal(res["traj_t"], c["traj_t"])
    perm_inv = np.argsort(c["perm"])
    U, V = res["U"][perm_inv], res["V"]
    if bool(c["transposed"]):
        U, V = V.T, U.T
    assert np.array_equal(U, c["U"]) and np.array_equal(V, c["V"])


def test_spec_worked_examples():
    # trop_matmul
    P, arg, _ = oracle.trop_matmul(np.array([[0., 1], [2, 3]]), np.array([[0., 1], [1, 0]]))
    assert P.tolist() == [[2, 1], [4, 3]]
    # masked_minplus (-U)^T (x)* R, U=[[0],[1]], R=[[2,3],[4,5]] -> [[2,3]]
    X = np.array([[2., 3], [4, 5]])
    M = np.ones((2, 2), bool)
    assert oracle.residuate_row(X, M, np.array([0., 1])).tolist() == [2, 3]
    M2 = M.copy(); M2[1, 0] = False
    assert oracle.residuate_row(X, M2, np.array([0., 1]))[0] == 2
    # b_norm [[1,-2],[missing,3]] -> 6; empty -> 0
    assert oracle.b_norm(np.array([1., -2, 3])) == 6 and oracle.b_norm(np.zeros(0)) == 0
    # approx_error example
    assert oracle.approx_error(X, M, np.array([[0.], [1]]), np.array([[2., 3]])) == 2
    M3 = M.copy(); M3[1, 1] = False
    assert oracle.approx_error(X, M3, np.array([[0.], [1]]), np.array([[2., 3]])) == 1
    # argmax tie -> smallest index
    _, a, _ = oracle.trop_matmul(np.array([[0., 0]]), np.array([[3.], [3.]]))
    assert a[0, 0] == 0
    _, a, _ = oracle.trop_matmul(np.array([[0., 1]]), np.array([[5.], [5.]]))
    assert a[0, 0] == 1
    # f_ulf 2x2 worked case
    U1, V1, f = oracle.f_ulf(X, M, np.array([[0.], [0]]), np.array([[2., 3]]), 1, 0, 0)
    assert U1.ravel().tolist() == [0, 2] and V1.ravel().tolist() == [2, 3] and f == 0
    with pytest.raises(ValueError):
        oracle.f_ulf(X, M2, np.array([[0.], [0]]), np.array([[2., 3]]), 1, 0, 0)
    # constant matrix: U all c, V all 0, error 0
    C = np.full((3, 4), 2.5)
    Vc = oracle.residuate_row(C, np.ones((3, 4), bool), np.full(3, 2.5))
    assert Vc.tolist() == [0, 0, 0, 0]


def test_f32_fit_properties():
    rng = np.random.default_rng(11)
    m, n, r = 24, 40, 3
    A = rng.random((m, r)); B = rng.random((r, n))
    X = (np.max(A[:, :, None] + B[None], axis=1) + rng.normal(0, 0.05, (m, n))).astype(np.float32)
    M = rng.random((m, n)) > 0.3
    M[:, 0] = True; M[0, :] = True
    U0 = X[:, rng.integers(0, n, r)].copy()
    U0[~np.isfinite(U0)] = 1
    U0 = U0.astype(np.float32)
    V0 = np.stack([oracle.residuate_row(X, M, U0[:, k]) for k in range(r)])
    a = oracle.fit(X, M, U0, V0, budget_sweeps=4, epsilon=0.0)
    b = oracle.fit(X, M, U0, V0, budget_sweeps=4, epsilon=0.0)
    assert np.array_equal(a["traj_err"], b["traj_err"]) and np.array_equal(a["U"], b["U"])
    e = a["traj_err"]
    assert np.all(np.diff(e) <= 0) and e[-1] < e[0]
    # subsolution U (x) V <= X on given entries, up to rounding
    P, _, _ = oracle.trop_matmul(a["U"], a["V"])
    assert np.all(P[M] <= X[M] + 1e-5)
    # the objective is the exact sum of the binary32 residuals
    res = np.abs(X[M] - P[M])
    assert a["traj_err"][-1] == math.fsum(res.astype(np.float64).tolist())
