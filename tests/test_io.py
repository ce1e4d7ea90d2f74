"""Matrix input/output, CPU only: the native CSV reader
against the reference's parsing rules (io.py:33-60, restated below as the checker),
the writer's round trip, and the binary masked-matrix format."""

import csv

import numpy as np
import pytest

import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import io as sio


def ref_load(path, has_header=False):
    """io.py:33-60: csv records, blank records skipped, cells stripped, "" / "nan" missing."""
    rows, masks = [], []
    with open(path, newline="") as fh:
        for idx, record in enumerate(csv.reader(fh)):
            if has_header and idx == 0:
                continue
            if not record:
                continue
            vals, given = [], []
            for cell in record:
                tok = cell.strip()
                if tok.lower() in {"", "nan"}:
                    vals.append(np.nan)
                    given.append(False)
                else:
                    vals.append(float(tok))
                    given.append(True)
            rows.append(vals)
            masks.append(given)
    if not rows:
        raise ValueError(f"{path}: no data rows")
    widths = {len(r) for r in rows}
    if len(widths) != 1:
        raise ValueError(f"{path}: ragged rows (widths {sorted(widths)})")
    return np.array(rows), np.array(masks)


def same(R, ref):
    vals, mask = ref
    return np.array_equal(R.mask, mask) and np.array_equal(R.values[mask], vals[mask])


def test_roundtrip_random(tmp_path):
    rng = np.random.default_rng(0)
    for t, (m, n) in enumerate([(1, 1), (5, 7), (40, 33), (300, 120)]):
        X = rng.normal(size=(m, n)) * 10.0 ** rng.integers(-8, 9, size=(m, n))
        M = rng.random((m, n)) < 0.7
        M[:, 0] = True
        M[0, :] = True
        R = pkg.MaskedMatrix(X, M)
        p = tmp_path / f"r{t}.csv"
        sio.save_matrix_csv(p, R, header=[f"c{j}" for j in range(n)] if t % 2 else None)
        L = sio.load_matrix_csv(p, has_header=bool(t % 2), threads=3)
        assert same(L, ref_load(p, bool(t % 2)))
        assert np.array_equal(L.values[M], X[M]) and np.array_equal(L.mask, M)


def test_reference_parsing_rules(tmp_path):
    text = 'h1,h2,h3\r\n 1.5 ,nan,\n\n"2.25",NaN,  -3e-5\n1_000,  ,7\n'
    p = tmp_path / "rules.csv"
    p.write_text(text)
    L = sio.load_matrix_csv(p, has_header=True)
    assert same(L, ref_load(p, True))
    assert L.shape == (3, 3)


@pytest.mark.parametrize("text,msg", [("1,2\n3\n", "ragged rows"), ("\n\n", "no data rows"),
                                      ("1,abc\n", "could not convert")])
def test_errors(tmp_path, text, msg):
    p = tmp_path / "bad.csv"
    p.write_text(text)
    with pytest.raises(ValueError, match=msg):
        ref_load(p)
    with pytest.raises(ValueError, match=msg):
        sio.load_matrix_csv(p)


def test_binary_format(tmp_path):
    from paper_2205_06619_b200 import gen
    for R in (gen.config1(), gen.config3(m=64, n=96, rank=3)):
        p = tmp_path / "m.bin"
        sio.save_matrix_bin(p, R)
        L = sio.load_matrix_bin(p)
        assert L.dtype == R.dtype and np.array_equal(L.mask, R.mask)
        assert np.array_equal(L.values[R.mask], R.values[R.mask])
        assert p.stat().st_size == 32 + (R.m * R.n + 7) // 8 + R.given_count * R.values.itemsize


def test_datagen_matches_reference():
    """SynthSpec / gen_mixture / apply_mask / gen_tall_wide_pair draw the reference's
    random numbers and reproduce its datasets (tests/golden/datagen.npz)."""
    from conftest import GOLDEN
    from paper_2205_06619_b200 import datagen
    g = np.load(f"{GOLDEN}/datagen.npz")
    for t, (r, c, lam, k, seed, frac) in enumerate(g["specs"]):
        spec = datagen.SynthSpec(int(r), int(c), float(lam), true_rank=int(k), seed=int(seed),
                                 mask_fraction=float(frac))
        R, A, B = datagen.gen_mixture(spec)
        assert np.array_equal(A, g[f"s{t}_A"]) and np.array_equal(B, g[f"s{t}_B"])
        assert np.array_equal(R, g[f"s{t}_R"])
        train, test = datagen.apply_mask(R, float(frac), seed=int(seed) + 100)
        assert np.array_equal(train.mask, g[f"s{t}_given"]) and np.array_equal(test, g[f"s{t}_test"])
        tall, wide = datagen.gen_tall_wide_pair(spec)
        assert np.array_equal(tall, g[f"s{t}_tall"]) and np.array_equal(wide, g[f"s{t}_wide"])
    with pytest.raises(ValueError):
        datagen.SynthSpec(2, 5, 0.5, true_rank=3)


def _traj(t, e, t_max):
    tr = pkg.Trajectory(t_init=0.0, t_max=t_max, time_unit="sweeps")
    for a, b in zip(t, e):
        tr.append(float(a), float(b))
    return tr


def test_host_statistics_match_reference():
    """metrics.py's trajectory statistics (tests/golden/hoststats.npz, from the reference)."""
    from conftest import GOLDEN
    from paper_2205_06619_b200 import metrics as M
    g = np.load(f"{GOLDEN}/hoststats.npz")
    base = _traj(g["base_t"], g["base_e"], 10.0)
    other = _traj(g["other_t"], g["other_e"], 10.0)
    assert np.array_equal(M.make_grid(10.0, 0.7), g["grid"])
    assert np.array_equal(M.make_grid(3.0, 1.0, 0.5), g["grid2"])
    assert np.array_equal(M.step_interpolate(base.times, base.errors, g["grid"]), g["interp"])
    assert np.array_equal(M.normalized_error(other, base, g["grid"]), g["ne"])
    assert np.array_equal(np.array(M.bootstrap_ci(g["samples"], n_resamples=300, level=0.9, seed=3)), g["ci"])
    assert np.array_equal(M.rank_methods(g["scores"]), g["ranks"])
    assert np.array_equal(M.rank_methods(g["scores"], lower_is_better=False), g["ranks_hi"])
    assert np.array_equal(M.average_ranks(g["ranks"]), g["avg"])
    assert np.array_equal(np.array([M.nemenyi_cd(4, 6), M.nemenyi_cd(3, 10, 0.1)]), g["cd"])
    ttr = [M.time_to_reach(base, float(base.errors[5]), g["grid"]), M.time_to_reach(base, -1.0, g["grid"])]
    assert np.array_equal(np.array(ttr), g["ttr"]) and ttr[1] == M.NEVER
    assert M.omega(g["samples"][:20], g["samples"][20:]) == float(g["omega"])


def test_sidecar_files_match_reference(tmp_path):
    """io.py's JSONL / JSON / CSV bundles: the same bytes as the reference's, and they
    read back (tests/golden/hoststats_files, from the reference)."""
    import filecmp
    from conftest import GOLDEN
    from paper_2205_06619_b200 import datagen
    ref = f"{GOLDEN}/hoststats_files"
    g = np.load(f"{GOLDEN}/hoststats.npz")
    base = _traj(g["base_t"], g["base_e"], 10.0)
    sio.save_trajectory(tmp_path / "traj.jsonl", base)
    assert filecmp.cmp(tmp_path / "traj.jsonl", f"{ref}/traj.jsonl", shallow=False)
    back = sio.load_trajectory(tmp_path / "traj.jsonl")
    assert back.times == base.times and back.errors == base.errors
    U = sio.load_matrix_csv(f"{ref}/p_U.csv").values
    V = sio.load_matrix_csv(f"{ref}/p_V.csv").values
    ori = pkg.Orientation(True, pkg.Permutation(np.array([1, 0])), None)
    sio.save_factors(tmp_path, pkg.FactorPair(U, V, 2, ori), config={"seed": 3, "method": "FastSTMF"}, prefix="p_")
    for f in ("p_U.csv", "p_V.csv", "p_factors.json"):
        assert filecmp.cmp(tmp_path / f, f"{ref}/{f}", shallow=False), f
    U2, V2, side = sio.load_factors(tmp_path, prefix="p_")
    assert np.array_equal(U2, U) and side["rank"] == 2
    ds = f"{ref}/ds"
    train, test_mask, test_values, meta = sio.load_dataset(ds)
    X = np.where(test_mask, test_values, train.values)
    A = sio.load_matrix_csv(f"{ds}/true_A.csv").values
    B = sio.load_matrix_csv(f"{ds}/true_B.csv").values
    tr2, te2 = datagen.apply_mask(X, 0.3, seed=2)
    assert np.array_equal(tr2.mask, train.mask) and np.array_equal(te2, test_mask)
    sio.save_dataset(tmp_path / "ds", tr2, te2, X, {"name": "toy", "lam": 0.5}, A=A, B=B)
    for f in ("dataset.json", "train.csv", "true_A.csv", "true_B.csv"):
        assert filecmp.cmp(tmp_path / "ds" / f, f"{ds}/{f}", shallow=False), f
