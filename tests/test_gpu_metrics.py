"""Device evaluation step: prediction rmse and (masked)
distance correlation, bit-identical to the reference's numpy expressions
(metrics.py:87-139, restated here as the checker)."""

import numpy as np
import pytest

import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import metrics

pytestmark = pytest.mark.gpu


def np_rmse(pred, truth, mask):  # metrics.py:87-95
    diff = (np.asarray(pred, np.float64) - np.asarray(truth, np.float64))[np.asarray(mask, bool)]
    return 0.0 if diff.size == 0 else float(np.sqrt(np.mean(diff ** 2)))


def np_cd(x):  # metrics.py:120-123
    d = np.abs(x[:, None] - x[None, :])
    return d - d.mean(axis=0)[None, :] - d.mean(axis=1)[:, None] + d.mean()


def np_dc(x, y):  # metrics.py:98-117
    A, B = np_cd(np.asarray(x, np.float64).ravel()), np_cd(np.asarray(y, np.float64).ravel())
    dvx, dvy = np.mean(A * A), np.mean(B * B)
    if dvx <= 0.0 or dvy <= 0.0:
        return 0.0
    return float(np.sqrt(max(np.mean(A * B), 0.0) / np.sqrt(dvx * dvy)))


def test_rmse_matches_numpy():
    rng = np.random.default_rng(1)
    for m, n, d in ((1, 1, 1.0), (7, 13, 0.5), (100, 200, 0.2), (300, 1000, 0.9), (64, 64, 0.0)):
        pred = rng.normal(size=(m, n))
        truth = rng.normal(size=(m, n)) * 3
        mask = rng.random((m, n)) < d
        assert metrics.rmse(pred, truth, mask) == np_rmse(pred, truth, mask), (m, n, d)


def test_prediction_rmse_of_a_fit():
    """The reference's evaluation flow: fit on the training mask, rmse of
    FactorPair.product() on the held-out entries."""
    from paper_2205_06619_b200 import gen
    R = gen.config1()
    full = np.where(R.mask, R.values, 0.0)
    rng = np.random.default_rng(4)
    test = R.mask & (rng.random(R.mask.shape) < 0.1)
    train = pkg.MaskedMatrix(R.values, R.mask & ~test)
    pair, _ = pkg.fast_stmf(train, 3, pkg.RunConfig(rank=3, budget_sweeps=2, epsilon=0.0, seed=42))
    P = pair.product()
    assert np.array_equal(P, np.max(pair.U[:, :, None] + pair.V[None, :, :], axis=1))
    assert metrics.rmse(P, full, test) == np_rmse(P, full, test)


def test_distance_correlation_matches_numpy():
    rng = np.random.default_rng(2)
    for n in (2, 3, 17, 129, 500, 2000):
        x = rng.normal(size=n)
        y = x * 0.5 + rng.normal(size=n) * 0.3
        assert metrics.distance_correlation(x, y) == np_dc(x, y), n
    assert metrics.distance_correlation(np.ones(5), np.arange(5.0)) == 0.0
    with pytest.raises(ValueError):
        metrics.distance_correlation([1.0], [2.0])


def test_masked_dc_subsamples_like_the_reference():
    rng = np.random.default_rng(3)
    truth = rng.normal(size=(80, 60))
    approx = truth + rng.normal(size=(80, 60)) * 0.2
    mask = rng.random((80, 60)) < 0.7
    x, y = truth[mask], approx[mask]
    idx = np.random.default_rng(0).choice(x.size, size=2000, replace=False)
    assert metrics.masked_dc(truth, approx, mask) == np_dc(x[idx], y[idx])
    assert metrics.masked_dc(truth, approx, mask, max_entries=10_000) == np_dc(x, y)


def test_b_norm_matches_reference(ops):
    """tropical.b_norm on the device: the reference's values on 30 arrays up to 200 K
    elements (tests/golden/ops.npz, bn*_w / bn_sums)."""
    for t in range(int(ops["n_bn"])):
        assert pkg.b_norm(ops[f"bn{t}_w"]) == float(ops["bn_sums"][t]), t
    assert pkg.b_norm(np.zeros((0,))) == 0.0


def test_td_helpers(ops):
    """td_grid (device product) and the single-entry / single-line helpers against the
    reference's td_grid column sums (ops.npz scores) and direct restatements."""
    for c in range(0, int(ops["n_ops"]), 2):
        X, M, U, V = (ops[f"c{c}_{k}"] for k in ("X", "M", "U", "V"))
        if not M.any(axis=0).all() or not M.any(axis=1).all():
            continue
        R = pkg.MaskedMatrix(X, M)
        grid = pkg.td_grid(R, U, V)
        assert np.array_equal(grid.sum(axis=0), ops[f"c{c}_scores"]), c
        gi, gj = np.nonzero(M)
        i, j = int(gi[0]), int(gj[0])
        assert pkg.td(R, U, V, i, j) == grid[i, j]
        assert pkg.argmax_k(U, V, i, j) == int(ops[f"c{c}_arg"][i, j])
        assert pkg.td_row(R, U, V, i) == float(np.sum(grid[i][M[i]]))
        assert pkg.td_col(R, U, V, j) == float(np.sum(grid[:, j][M[:, j]]))
