"""INTEGRATION.md §2 is runnable: integration/tropfact_b200.py binds a tropfact package
to libstmf_b200.so over ctypes and the C ABI alone, and its fast_stmf equals the
package's own fast_stmf bit for bit.  With the unmodified reference installed in
baseline/_ref (bench.py's reference arm) it runs against that; it always also runs
against this repository's mirror of the reference API."""

import importlib
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

pytestmark = pytest.mark.gpu
sys.path.insert(0, os.path.join(ROOT, "integration"))
import tropfact_b200  # noqa: E402

REF = os.path.join(ROOT, "baseline", "_ref")


def _packages():
    pk = [("mirror", "paper_2205_06619_b200")]
    if os.path.isdir(os.path.join(REF, "tropfact")):
        pk.append(("reference", "tropfact"))
    return pk


@pytest.mark.parametrize("which,name", _packages())
def test_binding_matches_package_fast_stmf(which, name):
    if which == "reference" and REF not in sys.path:
        sys.path.insert(0, REF)
    tf = importlib.import_module(name)
    from paper_2205_06619_b200 import gen
    C = gen.config1()
    X, M = C.values[:80, :60], C.mask[:80, :60]
    R = tf.MaskedMatrix(np.where(M, X, np.nan), M)
    cfg = tf.RunConfig(rank=3, budget_sweeps=3, epsilon=0.0, seed=11)
    pb, tb = tropfact_b200.fast_stmf(tf, R, 3, cfg)
    # the package's own fast_stmf (for the reference: the unmodified numpy code, 3 sweeps
    # of an 80 x 60 crop take seconds)
    pr, tr = tf.fast_stmf(R, 3, cfg)
    assert np.array_equal(pb.U, pr.U) and np.array_equal(pb.V, pr.V)
    assert tb.errors == tr.errors and tb.times == tr.times
