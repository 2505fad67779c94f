"""Reblurred (preconditioned) CGLS (config 2's "CGLS-type"
iteration).  Not in the reference, so the oracle (oracle.cgls) restates the
standard recurrence from the reference's primitives; parity of the recurrence
is unpinned.  CPU: recurrence properties of the oracle; GPU: the
device run against it."""
import numpy as np
import pytest


def _problem(n, name="C2"):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS[name]
    f, g, taps = cf.make_problem(c, n=n)
    return c, f, g, taps


def test_oracle_cgls_properties(oracle):
    c, f, g, taps = _problem(24)
    run = oracle.cgls(taps, g, f_true=f, max_iters=30)
    res = run["residual_history"]
    # the reblurred A' is not A^T under AR BCs, so ||r_k|| need not be monotone
    # (no CGLS optimality), but the data misfit drops
    assert res[-1] < res[0]
    # the residual recurrence equals g - A x_k
    run2 = oracle.cgls(taps, g, f_true=f, max_iters=30, stop=oracle.STOP_FIXED, fixed_iters=30)
    r = g - oracle.apply(taps, run2["restored"])
    assert abs(np.linalg.norm(r) - run2["residual_history"][-1]) <= 1e-8 * np.linalg.norm(g)
    # identity preconditioner reproduces plain CGLS
    ident = np.ones_like(g)
    run3 = oracle.cgls(taps, g, d=ident, f_true=f, max_iters=30)
    np.testing.assert_allclose(run3["residual_history"], res, rtol=1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("precond", [False, True])
@pytest.mark.parametrize("name,n,iters", [("C2", 64, 25), ("C1", 96, 20)])
def test_cgls_matches_oracle(dbx, oracle, precond, name, n, iters):
    dev = dbx
    c, f, g, taps = _problem(n, name)
    op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n)
    d = dev.build_tikhonov(dev.Psf(taps), dev.PreconditionerSpec(dev.Algebra.AntiReflective, c.alpha), n, n) \
        if precond else None
    run = dev.cgls(op, g, dev.SolverConfig(max_iters=iters, track_rre_against=f), d=d, keep_iterates=True)
    ref = oracle.cgls(taps, g, d=oracle.build_tikhonov(taps, c.alpha, n, n) if precond else None, f_true=f,
                      max_iters=iters, keep_iterates=True)
    assert run.iterations_executed == ref["iterations_executed"]
    assert run.best_iteration == ref["best_iteration"]
    for k in range(iters):
        e = np.linalg.norm(run.iterates[k] - ref["iterates"][k]) / np.linalg.norm(ref["iterates"][k])
        assert e <= 1e-10, (k + 1, e)
    np.testing.assert_allclose(run.residual_history, ref["residual_history"], rtol=1e-10, atol=0)
    np.testing.assert_allclose(run.rre_history, ref["rre_history"], rtol=1e-10, atol=0)


@pytest.mark.gpu
def test_cgls_batch_and_residual_rule(dbx, oracle):
    dev = dbx
    c, f, g, taps = _problem(48)
    B = 3
    gb = np.stack([g] * B)
    fb = np.stack([f] * B)
    op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, 48, 48, batch=B)
    runs = dev.cgls(op, gb, dev.SolverConfig(max_iters=15, track_rre_against=fb))
    for r in runs[1:]:
        assert r.residual_history == runs[0].residual_history
    full = oracle.cgls(taps, g, max_iters=40, stop=oracle.STOP_FIXED, fixed_iters=40)
    eps = 1.0000001 * min(full["residual_history"][:6]) / np.linalg.norm(g)
    stop = dev.StoppingRule.residual_below(eps)
    one = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, 48, 48)
    rr = dev.cgls(one, g, dev.SolverConfig(max_iters=40, stop=stop))
    ref = oracle.cgls(taps, g, max_iters=40, stop=oracle.STOP_RESID, resid_eps=eps)
    assert rr.iterations_executed == ref["iterations_executed"] <= 6
