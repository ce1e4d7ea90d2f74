"""Host-side logic of the drop-in API (CPU only): types, validation errors, method
parsing, orientation + Random-Acol draws (bit-equal to the reference's), the
config generators, and that the CUDA library loads and exports every symbol
declared in include/stmf_b200.h (no device calls)."""

import ctypes
import os
import re

import numpy as np
import pytest

import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import _ext, engine, gen
from conftest import ROOT, fit_case


def _has_gpu():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def header_symbols():
    src = open(os.path.join(ROOT, "include", "stmf_b200.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(stmf_\w+)\s*\(", src, re.M)))


def test_library_exports_header_symbols():
    _ext.build()
    L = ctypes.CDLL(_ext.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 15
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_ext.EXPORTED_SYMBOLS) == syms
    L.stmf_version.restype = ctypes.c_char_p
    assert b"sm_100a" in L.stmf_version()


def test_library_is_sm100a():
    out = os.popen(f"cuobjdump --list-elf {_ext.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_runconfig_validation():
    for bad in (dict(rank=0, budget_sweeps=1), dict(rank=1), dict(rank=1, budget_sweeps=-1),
                dict(rank=1, budget_seconds=0.0), dict(rank=1, budget_sweeps=1, acol_columns=0),
                dict(rank=1, budget_sweeps=1, epsilon=-1.0)):
        with pytest.raises(ValueError):
            pkg.RunConfig(**bad).validate()
    pkg.RunConfig(rank=2, budget_sweeps=0).validate()


def test_parse_method():
    assert pkg.parse_method("FastSTMF") == pkg.FASTSTMF
    assert pkg.parse_method("stmf_byrow_randpermr_td_a_w") == pkg.FASTSTMF
    assert pkg.parse_method("STMF") == pkg.BASELINE
    assert pkg.parse_method("STMF_ByRow_PermR_TD").prefer_wide is False
    with pytest.raises(ValueError):
        pkg.parse_method("nonsense")
    with pytest.raises(ValueError):
        pkg.StrategySpec("ByElement", "TD_A", "PermC")


def test_every_method_needs_the_device():
    """No CPU fallback: every fit method goes through the CUDA library."""
    if _has_gpu():
        pytest.skip("a CUDA device is present")
    R = pkg.MaskedMatrix(np.ones((3, 4)))
    cfg = pkg.RunConfig(rank=1, budget_sweeps=1)
    for meth in ("STMF", "STMF_ByMatrix_NoPerm_TD_W", "STMF_ByElement_PermC_TD", "STMF_ByRow_PermR_SEQ",
                 "FastSTMF"):
        with pytest.raises(_ext.StmfError):
            pkg.fit(R, 1, meth, cfg)


def test_validation_before_device_work():
    M = np.ones((3, 4), bool)
    M[1] = False
    R = pkg.MaskedMatrix(np.ones((3, 4)), M)
    with pytest.raises(ValueError, match="row 1 has no given entries"):
        pkg.fast_stmf(R, 1, pkg.RunConfig(rank=1, budget_sweeps=1))
    with pytest.raises(ValueError, match="set budget_sweeps"):
        pkg.fast_stmf(pkg.MaskedMatrix(np.ones((2, 2))), 1, pkg.RunConfig(rank=1))


def test_masked_matrix_and_orientation():
    X = np.arange(12.0).reshape(3, 4)
    M = X % 5 != 0
    R = pkg.MaskedMatrix(X, M)
    assert np.isnan(R.values[~M]).all() and R.given_count == M.sum()
    with pytest.raises(ValueError):
        pkg.MaskedMatrix(X, M[:2])
    p = pkg.Permutation(np.array([2, 0, 1]))
    assert np.array_equal(p.inverse[p.forward], np.arange(3))
    with pytest.raises(ValueError):
        pkg.Permutation(np.array([0, 0, 1]))
    ori = pkg.Orientation(True, pkg.Permutation(np.array([3, 1, 0, 2])), None)
    U = np.arange(8.0).reshape(4, 2)
    V = np.arange(6.0).reshape(2, 3)
    U2, V2 = ori.restore(U, V)
    assert U2.shape == (3, 2) and V2.shape == (2, 4)
    assert np.array_equal(V2, U[ori.row_perm.inverse].T)
    R32 = pkg.MaskedMatrix(X, M, dtype=np.float32)
    assert R32.dtype == np.float32 and R32.transpose().dtype == np.float32


@pytest.mark.parametrize("name", ["s0", "s1", "s2", "s3", "conv", "c1"])
def test_orientation_and_acol_draws_match_reference(fits, name):
    c = fit_case(fits, name)
    R = pkg.MaskedMatrix(c["R"], c["M"])
    rng = np.random.default_rng(int(c["seed"]))
    work, ori = engine._orient_faststmf(R, rng)
    assert ori.transposed == bool(c["transposed"])
    assert np.array_equal(ori.row_perm.forward, c["perm"])
    assert np.array_equal(work.mask, c["work_M"])
    assert np.array_equal(work.values[work.mask], c["work_X"][c["work_M"]])
    U0 = engine.acol_means(work, int(c["rank"]), 5, rng)
    assert np.array_equal(U0, c["U0"])


def test_config1_generator_matches_reference_datagen(fits):
    c = fit_case(fits, "c1")
    R = gen.config1()
    assert np.array_equal(R.mask, c["M"])
    assert np.array_equal(R.values[R.mask], c["R"][c["M"]])


def test_config4_generator_small_is_covered_and_blocked():
    R = gen.config4(seed=3, m=256, n=300, rank=4, blocks=4)
    R.validate_coverage()
    assert R.dtype == np.float32
    rates = 1 - R.mask.mean(axis=1)
    assert 0.8 < rates.mean() < 0.95  # Beta(9, 1) mean 0.9
    R2 = gen.config4(seed=3, m=256, n=300, rank=4, blocks=4)
    assert np.array_equal(R.mask, R2.mask) and np.array_equal(R.values[R.mask], R2.values[R2.mask])


def test_orientation_apply_factors_inverts_restore():
    import numpy as np
    from paper_2205_06619_b200.tropical import Permutation
    from paper_2205_06619_b200.types import Orientation
    rng = np.random.default_rng(0)
    U, V = rng.random((7, 3)), rng.random((3, 5))
    for tr in (False, True):
        rows = 5 if tr else 7
        cols = 7 if tr else 5
        o = Orientation(tr, Permutation.random(rows, rng), Permutation.random(cols, rng))
        Uw, Vw = o.apply_factors(U, V)
        assert Uw.shape == (rows, 3) and Vw.shape == (3, cols)
        U2, V2 = o.restore(Uw, Vw)
        assert np.array_equal(U2, U) and np.array_equal(V2, V)
