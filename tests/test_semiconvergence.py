"""semiconvergence_report (reference solver.hpp:152-160): the
first RRE minimum (std::min_element), its value, and the 5% divergence flag.
CPU: the product's host function against the oracle restatement on crafted
histories (ties, plateaus, monotone, the 5% edge, empty).  GPU: the report of
a device D-Landweber run equals the oracle run's report."""
import numpy as np
import pytest

from paper_1211_0393_b200 import RestorationRun, semiconvergence_report

CASES = [
    [0.5],                                   # one iteration
    [0.5, 0.4, 0.3, 0.2, 0.1],               # monotone: best = last, no divergence
    [0.5, 0.3, 0.2, 0.2, 0.25],              # tie: first minimum wins; 25% up
    [0.5, 0.3, 0.2, 0.21, 0.21],             # exactly +5%: strict >, not diverged
    [0.5, 0.3, 0.2, 0.2100001],              # just above 5%
    [0.3, 0.3, 0.3],                         # plateau from the start
    [1.0, 2.0, 3.0],                         # diverging from iteration 1
]


@pytest.mark.parametrize("hist", CASES)
def test_report_matches_oracle(oracle, hist):
    rep = semiconvergence_report(RestorationRun(rre_history=list(hist)))
    bi, br, dv = oracle.semiconvergence_report(hist)
    assert (rep.best_iter, rep.best_rre, rep.diverged_after) == (bi, br, dv)
    assert rep.best_iter == int(np.argmin(hist)) + 1


def test_empty_history_raises(oracle):
    with pytest.raises(ValueError, match="no RRE history"):
        semiconvergence_report(RestorationRun(rre_history=[]))
    with pytest.raises(ValueError, match="no RRE history"):
        oracle.semiconvergence_report([])


@pytest.mark.gpu
def test_report_of_device_run_matches_oracle_run(dbx, oracle):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C1"]
    n, iters = 96, 40
    f, g, taps = cf.make_problem(c, n=n)
    op = dbx.BlurOperator(dbx.Psf(taps), dbx.BoundaryCondition.AntiReflective, n, n)
    d = dbx.build_tikhonov(dbx.Psf(taps), dbx.PreconditionerSpec(dbx.Algebra.AntiReflective, c.alpha), n, n)
    cfg = dbx.SolverConfig(max_iters=iters, stop=dbx.StoppingRule.fixed(iters), track_rre_against=f)
    run = dbx.d_landweber(op, d, g, cfg)
    ref = oracle.landweber(taps, g, d=oracle.build_tikhonov(taps, c.alpha, n, n), f_true=f, max_iters=iters,
                           stop=oracle.STOP_FIXED, fixed_iters=iters)
    rep = semiconvergence_report(run)
    bi, br, dv = oracle.semiconvergence_report(ref["rre_history"])
    assert rep.best_iter == bi and rep.diverged_after == dv
    assert abs(rep.best_rre - br) <= 1e-10 * br
    assert rep.best_iter == run.best_iteration == ref["best_iteration"]
