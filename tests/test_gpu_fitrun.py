"""The reference's hand-driven protocol on the device: FitRun.try_ulf / try_urf / trial and
byrow_sweep / byrow_seq / byelement_sweep / bymatrix_step / bymatrix_candidates / select_k_*
(engine.py:240-310, strategies.py:147-314) replay the script of
tests/golden/make_golden_fitrun.py and must reproduce what the unmodified reference recorded:
every return value, the error after every step, the counters, the candidate lists, the
factors and the trajectory, bit for bit."""

import os

import numpy as np
import pytest

import paper_2205_06619_b200 as pkg
from paper_2205_06619_b200 import engine, strategies

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

# the same script as make_golden_fitrun.py (kept literal so the fixture pins it)
SCRIPT = ([("byrow", (i, "TD_A")) for i in range(0, 8)] + [("byrow", (i, "TD")) for i in range(8, 13)] +
          [("byrow", (i, "TD_B")) for i in range(13, 17)] + [("seq", 17), ("seq", 18), ("boundary", None),
                                                             ("byelement", None), ("boundary", None)] +
          [("bymatrix", None)] * 3 + [("byrow", (i, "SEQ")) for i in (19, 20)] + [("boundary", None)])


@pytest.fixture(scope="module")
def gold():
    return np.load(os.path.join(HERE, "golden", "fitrun.npz"))


def _matrix(gold):
    mask = gold["mask"]
    return pkg.MaskedMatrix(np.where(mask, gold["values"], np.nan), mask)


def test_selection_rules_and_trials(gold):
    R = _matrix(gold)
    U, V = gold["U0"].copy(), gold["V0"].copy()
    r = U.shape[1]
    probes = [tuple(p) for p in gold["probes"].tolist()]
    assert [strategies.select_k_td(U, V, i, j) for i, j in probes] == gold["sel_td"].tolist()
    assert [strategies.select_k_td_a(R, U, V, i, j) for i, j in probes] == gold["sel_td_a"].tolist()
    assert [strategies.select_k_td_b(R, U, V, i, j) for i, j in probes] == gold["sel_td_b"].tolist()
    cfg = pkg.RunConfig(rank=r, budget_sweeps=10, epsilon=0.0, seed=1)
    with engine.FitRun(R, U, V, cfg, wall_clock=False) as run:
        assert [run.trial(engine.f_ulf, i, j, (i + j) % r) for i, j in probes] == gold["trial_ulf"].tolist()
        assert [run.trial(engine.f_urf, i, j, (i + j) % r) for i, j in probes] == gold["trial_urf"].tolist()
        assert run.attempted_updates == 0 and np.array_equal(run.U, gold["U0"])  # trials record nothing
        cands = strategies.bymatrix_candidates(run)
        assert [[c.i, c.j, c.k] for c in cands] == gold["cand0"].tolist()
        assert [c.err_score for c in cands] == gold["cand0_score"].tolist()
        with pytest.raises(ValueError, match="missing"):
            i, j = np.argwhere(~R.mask)[0]
            run.try_ulf(int(i), int(j), 0)


def test_script_matches_reference(gold):
    R = _matrix(gold)
    U, V = gold["U0"].copy(), gold["V0"].copy()
    cfg = pkg.RunConfig(rank=U.shape[1], budget_sweeps=10, epsilon=0.0, seed=1)
    coin = np.random.default_rng(123)
    with engine.FitRun(R, U, V, cfg, wall_clock=False) as run:
        for step, (name, arg) in enumerate(SCRIPT):
            if name == "byrow":
                res = strategies.byrow_sweep(run, arg[0], arg[1])
            elif name == "seq":
                res = strategies.byrow_seq(run, arg)
            elif name == "byelement":
                res = strategies.byelement_sweep(run)
            elif name == "bymatrix":
                res = strategies.bymatrix_step(run, coin)
            else:
                run.current_sweep += 1
                res = run.mark_sweep_boundary()
            what = (step, name, arg)
            assert (-1 if res is None else int(res)) == gold["ret"][step], what
            assert run.err == gold["err"][step], what
            assert run.attempted_updates == gold["attempted"][step], what
            assert run.accepted_updates == gold["accepted"][step], what
        cands = strategies.bymatrix_candidates(run)
        assert [[c.i, c.j, c.k] for c in cands] == gold["cand1"].tolist()
        assert [c.err_score for c in cands] == gold["cand1_score"].tolist()
        assert np.array_equal(run.U, gold["U"]) and np.array_equal(run.V, gold["V"])
        assert U is run.U and np.array_equal(U, gold["U"])  # the caller's arrays, updated in place
        assert run.trajectory.times == gold["traj_t"].tolist()
        assert run.trajectory.errors == gold["traj_e"].tolist()
