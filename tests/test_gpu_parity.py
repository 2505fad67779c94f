"""GPU parity: the sm_100a path (through the C-ABI) against the CPU oracle on
identical seeded inputs.  Bars: operators <= 1e-12 relative L2, iterates
<= 1e-10 relative L2 at EVERY iteration (north_star), identical best-RRE
iteration, bit-identical reruns and batch-vs-single runs.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ITER_TOL = 1e-10   # north_star: relative L2 per iterate
OP_TOL = 1e-12     # single operator applications


def rel(a, b):
    a, b = np.asarray(a), np.asarray(b)
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def rand_psf(rng, q1, q2, sym=False):
    t = rng.uniform(0.05, 1.0, (2 * q1 + 1, 2 * q2 + 1))
    t /= t.sum()
    if sym:
        t = (t + t[::-1, :] + t[:, ::-1] + t[::-1, ::-1]) / 4.0
        t /= t.sum()
    return t


@pytest.fixture(scope="module")
def dev(dbx):
    if dbx.lib().dbx_device_count() < 1:
        pytest.fail("no sm_100 device visible: GPU tests must run on a B200")
    return dbx


@pytest.mark.parametrize("n1,n2,q1,q2", [(7, 8, 1, 2), (24, 30, 1, 9), (37, 53, 3, 5), (64, 64, 7, 7),
                                         (100, 70, 0, 4), (3, 5, 1, 3), (130, 67, 15, 2)])
def test_blur_matches_oracle(dev, oracle, n1, n2, q1, q2):
    rng = np.random.default_rng(n1 * 1000 + n2 * 10 + q1)
    t = rand_psf(rng, q1, q2)
    f = rng.uniform(0, 1, (n1, n2))
    op = dev.BlurOperator(dev.Psf(t), dev.BoundaryCondition.AntiReflective, n1, n2)
    for adj in (False, True):
        got = dev.apply_reblur_adjoint(op, f) if adj else dev.apply(op, f)
        want = oracle.apply(t, f, adjoint=adj, path=1)
        assert rel(got, want) <= OP_TOL, (adj, rel(got, want))


def sep_psf(rng, q1, q2):
    """Rank-1 mask (outer product of two positive profiles), normalised."""
    a = rng.uniform(0.05, 1.0, 2 * q1 + 1)
    b = rng.uniform(0.05, 1.0, 2 * q2 + 1)
    t = np.outer(a, b)
    return t / t.sum()


@pytest.mark.parametrize("n1,n2,q1,q2,bc", [(64, 64, 7, 7, "ar"), (96, 130, 15, 4, "ar"), (200, 77, 7, 12, "ar"),
                                            (1024, 1024, 15, 15, "ar"), (61, 90, 15, 15, "reflective"),
                                            (40, 33, 7, 0, "ar"), (40, 2100, 7, 15, "ar"),
                                            (33, 1030, 15, 7, "ar"), (35, 1031, 15, 15, "reflective")])
def test_separable_column_pass_matches_oracle(dev, oracle, n1, n2, q1, q2, bc):
    """Rank-1 masks with q1, q2 in {7, 15} run the direct separable blur
    (rows_sep_seg: 1024-column row segments with their extension halo, then
    cols_sep_real); other rank-1 masks run the separable column pass inside
    the FFT engine (conv_col_sep: direct 2 q1 + 1 tap correlation of the
    extended column x one complex scale per column).  n2 = 2100 / 1030 / 1031
    span several row segments, the last shorter than q2 (its extension reads
    the previous segment).  A and A' match the oracle's full-mask correlation
    like the dense kernel spectrum does."""
    rng = np.random.default_rng(n1 * 7 + n2 * 3 + q1 + q2)
    t = sep_psf(rng, q1, q2)
    f = rng.uniform(0, 1, (n1, n2))
    BC = dev.BoundaryCondition.AntiReflective if bc == "ar" else dev.BoundaryCondition.Reflective
    obc = oracle.BC_ANTIREFLECTIVE if bc == "ar" else oracle.BC_REFLECTIVE
    for eng in (dev.ConvEngine.Fft, dev.ConvEngine.FftDense):
        op = dev.BlurOperator(dev.Psf(t), BC, n1, n2).set_conv(eng)
        sep, resid = op.separable()
        assert sep == (eng == dev.ConvEngine.Fft), (eng, sep, resid)
        assert resid <= 1e-14
        for adj in (False, True):
            got = dev.apply_reblur_adjoint(op, f) if adj else dev.apply(op, f)
            want = oracle.apply(t, f, adjoint=adj, path=1, bc=obc)
            assert rel(got, want) <= OP_TOL, (eng, adj, rel(got, want))


def test_separable_detection(dev):
    """The BASELINE's axis-aligned Gaussians (C1, C3, C5) factor at rounding
    level; the rotated (C4) and motion (C2) masks and a random mask do not."""
    from paper_1211_0393_b200 import configs as cf
    for name, want in (("C1", True), ("C3", True), ("C5", True), ("C2", False), ("C4", False)):
        c = cf.CONFIGS[name]
        taps = cf.make_psf(c)
        n = 256 if name != "C4" else 200
        op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n)
        sep, resid = op.separable()
        assert sep == (want and c.q in (7, 15)), (name, sep, resid)
    rng = np.random.default_rng(5)
    op = dev.BlurOperator(dev.Psf(rand_psf(rng, 15, 15)), dev.BoundaryCondition.AntiReflective, 128, 128)
    assert op.separable()[0] is False


@pytest.mark.parametrize("name,n", [("C1", 256), ("C2", 512), ("C3", 160), ("C4", 200), ("C5", 96)])
def test_config_blur_matches_oracle(dev, oracle, name, n):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS[name]
    f, g, taps = cf.make_problem(c, n=n)
    op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n)
    assert rel(dev.apply(op, f), oracle.apply(taps, f)) <= OP_TOL
    assert rel(dev.apply_reblur_adjoint(op, g), oracle.apply(taps, g, adjoint=True)) <= OP_TOL


@pytest.mark.parametrize("n1,n2", [(3, 3), (6, 7), (16, 16), (33, 20), (256, 256), (512, 300)])
def test_tensor_apply_matches_oracle(dev, oracle, n1, n2):
    rng = np.random.default_rng(n1 + 7 * n2)
    x = rng.uniform(-1, 1, (n1, n2))
    for kind in (dev.TransformKind.SineI, dev.TransformKind.AntiReflective,
                 dev.TransformKind.AntiReflectiveInverse):
        got = dev.tensor_apply(kind, x)
        want = oracle.tensor_apply(int(kind), x)
        assert rel(got, want) <= OP_TOL, (kind, rel(got, want))


@pytest.mark.parametrize("n1,n2,q1,q2,alpha", [(6, 7, 1, 1, 0.02), (16, 16, 2, 1, 0.05), (64, 48, 5, 3, 0.01),
                                               (256, 256, 7, 7, 0.02)])
def test_precondition_matches_oracle(dev, oracle, n1, n2, q1, q2, alpha):
    rng = np.random.default_rng(q1 * 31 + n1)
    t = rand_psf(rng, q1, q2)
    d = dev.build_tikhonov(dev.Psf(t), dev.PreconditionerSpec(dev.Algebra.AntiReflective, alpha), n1, n2)
    dref = oracle.build_tikhonov(t, alpha, n1, n2)
    assert rel(d.eigs, dref) <= 1e-14
    r = rng.uniform(-1, 1, (n1, n2))
    assert rel(dev.precondition_apply(d, r), oracle.precondition_apply(dref, r)) <= OP_TOL


def _trajectory_check(gpu_run, ref):
    assert gpu_run.iterations_executed == ref["iterations_executed"]
    assert gpu_run.best_iteration == ref["best_iteration"]
    for k in range(ref["iterations_executed"]):
        e = rel(gpu_run.iterates[k], ref["iterates"][k])
        assert e <= ITER_TOL, (k + 1, e)
    np.testing.assert_allclose(gpu_run.residual_history, ref["residual_history"], rtol=1e-10, atol=0)
    if len(ref["rre_history"]):
        np.testing.assert_allclose(gpu_run.rre_history, ref["rre_history"], rtol=1e-10, atol=0)
    assert rel(gpu_run.restored, ref["restored"]) <= ITER_TOL


@pytest.mark.parametrize("precond", [True, False])
def test_config1_full_trajectory(dev, oracle, precond):
    """C1 at full size: 256^2, q=7, 50 iterations, every iterate checked."""
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C1"]
    f, g, taps = cf.make_problem(c)
    op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, c.n, c.n)
    cfg = dev.SolverConfig(tau=1.0, max_iters=c.iters, track_rre_against=f)
    if precond:
        d = dev.build_tikhonov(dev.Psf(taps), dev.PreconditionerSpec(dev.Algebra.AntiReflective, c.alpha), c.n, c.n)
        run = dev.d_landweber(op, d, g, cfg, keep_iterates=True)
        ref = oracle.landweber(taps, g, d=oracle.build_tikhonov(taps, c.alpha, c.n, c.n), f_true=f,
                               max_iters=c.iters, keep_iterates=True)
    else:
        run = dev.landweber(op, g, cfg, keep_iterates=True)
        ref = oracle.landweber(taps, g, f_true=f, max_iters=c.iters, keep_iterates=True)
    _trajectory_check(run, ref)
    # below the reference's q > 7 cutover AUTO still picks the FFT engine here:
    # it unlocks the fused preconditioned pipeline for this shape
    assert op.engines()[0] == dev.ConvEngine.Fft
    assert op.pipeline_fused() == precond


@pytest.mark.parametrize("name,n,iters", [("C2", 128, 30), ("C3", 128, 20), ("C4", 160, 10), ("C5", 128, 10)])
def test_config_trajectories_scaled(dev, oracle, name, n, iters):
    """Configs' masks / noise / alpha on a reduced FOV the oracle finishes quickly.
    The oracle uses the reference's FFT correlation for q > 7 (blur.hpp:79-82)."""
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS[name]
    f, g, taps = cf.make_problem(c, n=n)
    op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n)
    d = dev.build_tikhonov(dev.Psf(taps), dev.PreconditionerSpec(dev.Algebra.AntiReflective, c.alpha), n, n)
    cfg = dev.SolverConfig(max_iters=iters, track_rre_against=f)
    run = dev.d_landweber(op, d, g, cfg, keep_iterates=True)
    ref = oracle.landweber(taps, g, d=oracle.build_tikhonov(taps, c.alpha, n, n), f_true=f, max_iters=iters,
                           keep_iterates=True)
    _trajectory_check(run, ref)
    if c.plain_too:
        run = dev.landweber(op, g, cfg, keep_iterates=True)
        ref = oracle.landweber(taps, g, f_true=f, max_iters=iters, keep_iterates=True)
        _trajectory_check(run, ref)


def test_batch_equals_single_and_deterministic(dev):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C3"]
    F, G, taps = cf.make_batch(c, 3, n=96)
    d = dev.build_tikhonov(dev.Psf(taps), dev.PreconditionerSpec(dev.Algebra.AntiReflective, c.alpha), 96, 96)
    opb = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, 96, 96, batch=3)
    runs = dev.d_landweber(opb, d, G, dev.SolverConfig(max_iters=12, track_rre_against=F))
    runs2 = dev.d_landweber(opb, d, G, dev.SolverConfig(max_iters=12, track_rre_against=F))
    op1 = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, 96, 96)
    for i in range(3):
        one = dev.d_landweber(op1, d, G[i], dev.SolverConfig(max_iters=12, track_rre_against=F[i]))
        assert np.array_equal(one.restored, runs[i].restored)
        assert one.rre_history == runs[i].rre_history
        assert one.residual_history == runs[i].residual_history
        assert runs2[i].rre_history == runs[i].rre_history
        assert np.array_equal(runs2[i].restored, runs[i].restored)


@pytest.mark.parametrize("name,n,chunks", [("C3", 1024, (2, 1, 1)), ("C1", 96, (1, 3))])
def test_chunked_host_run_equals_batch(dev, name, n, chunks):
    """dbx_landweber_run_chunks (copy/compute-overlapped host batch) equals
    the one-plan batch run bit for bit, fused (C3 full size) and separate-pass
    (C1 direct stencil) pipelines, plain pinned and pageable host arrays."""
    import torch
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS[name]
    B = sum(chunks)
    F, G, taps = cf.make_batch(c, B, n=n)
    spec = dev.PreconditionerSpec(dev.Algebra.AntiReflective, c.alpha)
    d = dev.build_tikhonov(dev.Psf(taps), spec, n, n)
    cfg = dev.SolverConfig(max_iters=4, track_rre_against=F)
    opb = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n, batch=B)
    ref = dev.d_landweber(opb, d, G, cfg)
    ops = [dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n, batch=k) for k in chunks]
    for pinned in (True, False):
        g = torch.from_numpy(G).pin_memory() if pinned else G
        fcfg = dev.SolverConfig(max_iters=4, track_rre_against=torch.from_numpy(F).pin_memory() if pinned else F)
        runs = dev.landweber_chunks(ops, g, fcfg, d=d)
        for i in range(B):
            assert np.array_equal(np.asarray(runs[i].restored), ref[i].restored)
            assert runs[i].rre_history == ref[i].rre_history
            assert runs[i].residual_history == ref[i].residual_history
            assert runs[i].best_iteration == ref[i].best_iteration
    with pytest.raises(ValueError):
        dev.landweber_chunks(ops, torch.from_numpy(G).cuda(), cfg, d=d)


def test_stopping_rules_and_errors(dev, oracle):
    rng = np.random.default_rng(383)
    n = 20
    t = 0.4 * rand_psf(rng, 1, 1, sym=True)
    t[1, 1] += 0.6
    f = rng.uniform(1, 2, (n, n))
    op = dev.BlurOperator(dev.Psf(t), dev.BoundaryCondition.AntiReflective, n, n)
    g = dev.apply(op, f)
    # residual rule (solver_test.cpp:96-109)
    run = dev.landweber(op, g, dev.SolverConfig(max_iters=500, stop=dev.StoppingRule.residual_below(1e-3)))
    ref = oracle.landweber(t, g, max_iters=500, stop=oracle.STOP_RESID, resid_eps=1e-3)
    assert run.iterations_executed == ref["iterations_executed"] < 500
    assert run.residual_history[-1] / np.linalg.norm(g) < 1e-3
    # fixed(0) returns the zero start (solver_test.cpp:27-39)
    run0 = dev.landweber(op, g, dev.SolverConfig(stop=dev.StoppingRule.fixed(0), track_rre_against=g))
    assert run0.iterations_executed == 0 and np.abs(run0.restored).max() == 0.0 and run0.rre_history == []
    # divergence guard (solver_test.cpp:85-94)
    opd = dev.BlurOperator(dev.delta_psf(1, 1), dev.BoundaryCondition.AntiReflective, 8, 8)
    with pytest.raises(dev.SolverDivergence):
        dev.landweber(opd, rng.uniform(1, 2, (8, 8)), dev.SolverConfig(tau=3.0, max_iters=200,
                                                                       stop=dev.StoppingRule.fixed(200)))
    with pytest.raises(ValueError):
        dev.landweber(op, g, dev.SolverConfig(tau=0.0))
    with pytest.raises(ValueError):
        dev.apply(op, np.ones((n, n + 1)))


def test_delta_mask_first_iterate(dev):
    """solver_test.cpp:133-150: AR D-Landweber with a delta mask: x1 = g/(1+alpha)."""
    rng = np.random.default_rng(397)
    n = 8
    g = rng.uniform(1, 2, (n, n))
    op = dev.BlurOperator(dev.delta_psf(), dev.BoundaryCondition.AntiReflective, n, n)
    for alpha, want in ((0.25, g / 1.25), (0.0, g)):
        d = dev.build_tikhonov(dev.delta_psf(), dev.PreconditionerSpec(dev.Algebra.AntiReflective, alpha), n, n)
        run = dev.d_landweber(op, d, g, dev.SolverConfig(max_iters=1, stop=dev.StoppingRule.fixed(1)))
        assert np.abs(run.restored - want).max() <= 1e-12


def test_identity_filter_reproduces_plain(dev):
    """solver_test.cpp:111-131 (AR variant): d == 1 gives the plain trajectory."""
    rng = np.random.default_rng(389)
    n = 12
    t = rand_psf(rng, 1, 1)
    f = rng.uniform(1, 2, (n, n))
    op = dev.BlurOperator(dev.Psf(t), dev.BoundaryCondition.AntiReflective, n, n)
    g = dev.add_noise(dev.apply(op, f), dev.NoiseSpec(0.001, 7))
    ident = dev.filter_from_eigs(np.ones((n, n)))
    cfg = dev.SolverConfig(max_iters=100, stop=dev.StoppingRule.fixed(100), track_rre_against=f)
    a = dev.landweber(op, g, cfg)
    b = dev.d_landweber(op, ident, g, cfg)
    np.testing.assert_allclose(a.rre_history, b.rre_history, rtol=0, atol=1e-12)
    assert np.abs(a.restored - b.restored).max() <= 1e-12


@pytest.mark.parametrize("name", ["C4", "C5"])
def test_full_size_properties(dev, name):
    """Size-independent properties at the BASELINE FOV (oracle too slow here):
    A maps a linear ramp to the ramp shifted by the mask's first moment (AR
    extension is exact on affine images), D with d == 1 is the identity
    (T T~ = I), and A is linear."""
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS[name]
    n = c.n
    taps = cf.make_psf(c)
    op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n)
    i = np.arange(n, dtype=np.float64)
    ramp = 0.3 + 1e-3 * i[:, None] - 2e-3 * i[None, :]
    s = np.arange(-c.q, c.q + 1, dtype=np.float64)
    m1 = float((taps.sum(axis=1) * s).sum())  # sum h(s1,s2) s1
    m2 = float((taps.sum(axis=0) * s).sum())
    want = 0.3 + 1e-3 * (i[:, None] - m1) - 2e-3 * (i[None, :] - m2)
    assert rel(dev.apply(op, ramp), want) <= 1e-12
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, (n, n))
    y = rng.uniform(0, 1, (n, n))
    assert rel(dev.apply(op, 2.0 * x - y), 2.0 * dev.apply(op, x) - dev.apply(op, y)) <= 1e-13
    ident = dev.filter_from_eigs(np.ones((n, n)))
    assert rel(dev.precondition_apply(ident, x), x) <= 1e-11


# ---------------------------------------------------------------------------
# engine coverage: FFT correlation vs direct stencil, Bluestein vs dense DST
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("n1,n2,q1,q2", [(24, 30, 1, 9), (64, 64, 7, 7), (100, 70, 8, 3), (130, 67, 15, 2),
                                         (200, 200, 31, 31), (37, 53, 3, 5), (5, 9, 1, 3)])
def test_fft_conv_engine_matches_oracle(dev, oracle, n1, n2, q1, q2):
    rng = np.random.default_rng(7 * n1 + n2 + q1)
    t = rand_psf(rng, q1, q2)
    f = rng.uniform(0, 1, (n1, n2))
    op = dev.BlurOperator(dev.Psf(t), dev.BoundaryCondition.AntiReflective, n1, n2).set_conv(dev.ConvEngine.Fft)
    assert op.engines()[0] == dev.ConvEngine.Fft
    for adj in (False, True):
        got = dev.apply_reblur_adjoint(op, f) if adj else dev.apply(op, f)
        assert rel(got, oracle.apply(t, f, adjoint=adj, path=2)) <= OP_TOL
        assert rel(got, oracle.apply(t, f, adjoint=adj, path=1)) <= OP_TOL


@pytest.mark.parametrize("n1,n2", [(3, 3), (6, 7), (16, 16), (33, 20), (256, 256), (512, 300), (1024, 1024)])
@pytest.mark.parametrize("engine", ["Fft", "Dense"])
def test_dst_engines_match_oracle(dev, oracle, n1, n2, engine):
    rng = np.random.default_rng(n1 + 3 * n2)
    x = rng.uniform(-1, 1, (n1, n2))
    eng = getattr(dev.DstEngine, engine)
    for kind in (dev.TransformKind.SineI, dev.TransformKind.AntiReflective,
                 dev.TransformKind.AntiReflectiveInverse):
        got = dev.tensor_apply(kind, x, engine=eng)
        assert rel(got, oracle.tensor_apply(int(kind), x)) <= OP_TOL, (kind, engine)
    t = rand_psf(rng, 2, 1)
    d = dev.build_tikhonov(dev.Psf(t), dev.PreconditionerSpec(dev.Algebra.AntiReflective, 0.02), n1, n2) \
        if min(n1, n2) >= 5 else None
    if d is not None:
        r = rng.uniform(-1, 1, (n1, n2))
        ref = oracle.precondition_apply(oracle.build_tikhonov(t, 0.02, n1, n2), r)
        assert rel(dev.precondition_apply(d, r, engine=eng), ref) <= OP_TOL


@pytest.mark.parametrize("n1,n2", [(116, 116), (116, 40), (2048, 64), (64, 2048), (114, 116)])
def test_pfa_dst_matches_oracle(dev, oracle, n1, n2):
    """Prime-factor core (N = 23 x 5 = 115, 23 x 89 = 2047 for C4: Good-Thomas
    rows of 23 in registers, Rader columns over the in-place CT core) against
    the oracle: tensor_apply along both axes (the column pass runs the
    transposed images through the same row kernel), the preconditioner
    (fused T~ d^T T pass) and SineI at N = n+1 = 115."""
    rng = np.random.default_rng(n1 * 7 + n2)
    x = rng.uniform(-1, 1, (n1, n2))
    kinds = [dev.TransformKind.AntiReflective, dev.TransformKind.AntiReflectiveInverse, dev.TransformKind.SineI]
    for kind in kinds:
        got = dev.tensor_apply(kind, x)
        assert rel(got, oracle.tensor_apply(int(kind), x)) <= OP_TOL, kind
    t = rand_psf(rng, 2, 2)
    d = dev.build_tikhonov(dev.Psf(t), dev.PreconditionerSpec(dev.Algebra.AntiReflective, 0.02), n1, n2)
    r = rng.uniform(-1, 1, (n1, n2))
    ref = oracle.precondition_apply(oracle.build_tikhonov(t, 0.02, n1, n2), r)
    assert rel(dev.precondition_apply(d, r), ref) <= OP_TOL


@pytest.mark.parametrize("n1,n2,kinds", [
    (24, 128, ("AntiReflective", "AntiReflectiveInverse")),  # N = n-1 = 23, 127 (prime; M = 22, 126)
    (22, 126, ("SineI",)),                                    # N = n+1 = 23, 127
])
def test_rader_dst_matches_oracle(dev, oracle, n1, n2, kinds):
    """Rader core of the packed DST (prime N, cyclic convolution of length
    N-1) forced at small sizes; AUTO selects it for C5 (N = 8191)."""
    rng = np.random.default_rng(n1 * 5 + n2)
    x = rng.uniform(-1, 1, (n1, n2))
    for name in kinds:
        kind = getattr(dev.TransformKind, name)
        got = dev.tensor_apply(kind, x, engine=dev.DstEngine.Rader)
        assert rel(got, oracle.tensor_apply(int(kind), x)) <= OP_TOL, name
    if "AntiReflective" in kinds:
        t = rand_psf(rng, 2, 3)
        d = dev.build_tikhonov(dev.Psf(t), dev.PreconditionerSpec(dev.Algebra.AntiReflective, 0.02), n1, n2)
        r = rng.uniform(-1, 1, (n1, n2))
        ref = oracle.precondition_apply(oracle.build_tikhonov(t, 0.02, n1, n2), r)
        assert rel(dev.precondition_apply(d, r, engine=dev.DstEngine.Rader), ref) <= OP_TOL


@pytest.mark.parametrize("n1,n2", [(25, 17), (9, 10), (257, 129), (65, 64)])
def test_packed_dst_even_n_matches_oracle(dev, oracle, n1, n2):
    """Odd image sizes (even DFT length N = n-1) run the packed FFT form too
    (formerly dense only)."""
    rng = np.random.default_rng(n1 * 3 + n2)
    x = rng.uniform(-1, 1, (n1, n2))
    for kind in (dev.TransformKind.SineI, dev.TransformKind.AntiReflective,
                 dev.TransformKind.AntiReflectiveInverse):
        got = dev.tensor_apply(kind, x, engine=dev.DstEngine.Fft)
        assert rel(got, oracle.tensor_apply(int(kind), x)) <= OP_TOL, kind


@pytest.mark.parametrize("name,n,iters,conv", [("C1", 256, 8, "Fft"), ("C2", 512, 5, "Auto"), ("C3", 1024, 3, "Auto")])
@pytest.mark.parametrize("fusion", [True, False])
def test_fused_pipeline_full_size(dev, oracle, name, n, iters, conv, fusion):
    """The fused row pipelines (fused.cu) at the compiled full-size shapes:
    C1 (conv 270, direct DST 255), C2 (conv 540, Bluestein 1024), C3 (conv
    1080, direct DST 1023); fused and unfused must both match the oracle."""
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS[name]
    f, g, taps = cf.make_problem(c, n=n)
    op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n)
    op.set_conv(getattr(dev.ConvEngine, conv)).set_fusion(fusion)
    d = dev.build_tikhonov(dev.Psf(taps), dev.PreconditionerSpec(dev.Algebra.AntiReflective, c.alpha), n, n)
    run = dev.d_landweber(op, d, g, dev.SolverConfig(max_iters=iters, track_rre_against=f), keep_iterates=True)
    ref = oracle.landweber(taps, g, d=oracle.build_tikhonov(taps, c.alpha, n, n), f_true=f, max_iters=iters,
                           keep_iterates=True)
    _trajectory_check(run, ref)


@pytest.mark.parametrize("conv,dst", [("Direct", "Dense"), ("Fft", "Fft"), ("Direct", "Fft"), ("Fft", "Dense")])
def test_engine_combinations_same_trajectory(dev, oracle, conv, dst):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C3"]
    n, iters = 96, 12
    f, g, taps = cf.make_problem(c, n=n)
    op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n)
    op.set_conv(getattr(dev.ConvEngine, conv)).set_dst(getattr(dev.DstEngine, dst))
    d = dev.build_tikhonov(dev.Psf(taps), dev.PreconditionerSpec(dev.Algebra.AntiReflective, c.alpha), n, n)
    run = dev.d_landweber(op, d, g, dev.SolverConfig(max_iters=iters, track_rre_against=f), keep_iterates=True)
    ref = oracle.landweber(taps, g, d=oracle.build_tikhonov(taps, c.alpha, n, n), f_true=f, max_iters=iters,
                           keep_iterates=True)
    _trajectory_check(run, ref)
