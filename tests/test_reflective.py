"""Reflective boundary conditions with the CosineIII (DCT-III) algebra — the
paper's comparison path.  CPU: the oracle's reflective
branch pinned to numpy/scipy re-derivations and the reference's own
assertions (boundary_test, spectral_test EigReflective, oracles_test
Dct3Structure); GPU: the device path against the oracle."""
import numpy as np
import pytest
import scipy.fft as sfft

REFL = 2


def rand_sym_psf(rng, q1, q2):
    t = rng.uniform(0.1, 1.0, (2 * q1 + 1, 2 * q2 + 1))
    t = (t + t[::-1, :] + t[:, ::-1] + t[::-1, ::-1]) / 4
    return t / t.sum()


def rand_psf(rng, q1, q2):
    t = rng.uniform(0.0, 1.0, (2 * q1 + 1, 2 * q2 + 1))
    return t / t.sum()


def numpy_blur(taps, f):
    """pad (boundary.hpp:49-55, numpy 'symmetric' = f_{-i} = f_{i-1}) + valid
    correlation with the rotated mask (g_i = sum_s h_s f_{i-s}, blur.hpp:48)."""
    q1, q2 = (taps.shape[0] - 1) // 2, (taps.shape[1] - 1) // 2
    P = np.pad(f, ((q1, q1), (q2, q2)), mode="symmetric")
    n1, n2 = f.shape
    g = np.zeros_like(f)
    for s1 in range(-q1, q1 + 1):
        for s2 in range(-q2, q2 + 1):
            g += taps[q1 + s1, q2 + s2] * P[q1 - s1:q1 - s1 + n1, q2 - s2:q2 - s2 + n2]
    return g


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_oracle_reflective_blur_matches_numpy(oracle):
    rng = np.random.default_rng(11)
    for (n1, n2, q1, q2) in [(6, 7, 1, 2), (12, 9, 3, 4), (20, 24, 9, 8)]:
        t = rand_psf(rng, q1, q2)
        f = rng.uniform(size=(n1, n2))
        want = numpy_blur(t, f)
        for path in (1, 2):
            assert rel(oracle.apply(t, f, path=path, bc=REFL), want) <= 1e-13
        # A' = blur with the 180-rotated mask (blur.hpp:87-90)
        assert rel(oracle.apply(t, f, adjoint=True, path=1, bc=REFL), numpy_blur(t[::-1, ::-1], f)) <= 1e-13
    # support: q <= n allowed, q > n rejected (boundary_test.cpp:48-53)
    f = np.ones((4, 4))
    oracle.apply(np.full((9, 9), 1 / 81), f, bc=REFL)
    with pytest.raises(ValueError):
        oracle.apply(np.full((1, 11), 1 / 11), f, bc=REFL)


def test_oracle_cosine3_matches_scipy(oracle):
    rng = np.random.default_rng(5)
    for m in (1, 2, 5, 16, 33, 256):
        v = rng.uniform(-1, 1, m)
        assert np.abs(oracle.cosine3_forward(v) - sfft.dct(v, type=2, norm="ortho")).max() <= 1e-14
        assert np.abs(oracle.cosine3_forward(v, inverse=True) - sfft.dct(v, type=3, norm="ortho")).max() <= 1e-14
    x = rng.uniform(size=(7, 10))
    want = sfft.dct(sfft.dct(x, type=2, norm="ortho", axis=0), type=2, norm="ortho", axis=1)
    assert rel(oracle.tensor_apply(1, x), want) <= 1e-14


def test_oracle_eig_reflective(oracle):
    # delta mask: all ones; random symmetric mask: lambda(0,0) = mask sum (spectral_test.cpp:15-22)
    d = oracle.build_tikhonov(np.ones((3, 3)) * 0 + np.eye(3)[1:2].T @ np.eye(3)[1:2], 0.0, 6, 5, bc=REFL)
    assert np.abs(d - 1.0).max() <= 1e-15
    rng = np.random.default_rng(157)
    p = rand_sym_psf(rng, 2, 2)
    n = 8
    lam = 1.0 / np.sqrt(oracle.build_tikhonov(p, 0.0, n, n, bc=REFL))  # |lambda| from d = 1/lambda^2
    # multiset of |eigenvalues| = dense eigenvalues of the reflective blur (spectral_test.cpp:24-33)
    A = np.column_stack([oracle.apply(p, e.reshape(n, n), path=1, bc=REFL).ravel() for e in np.eye(n * n)])
    dense = np.sort(np.abs(np.linalg.eigvals(A).real))
    assert np.abs(np.sort(lam.ravel()) - dense).max() <= 1e-8
    # Dct3Structure (oracles_test.cpp:118-129): A = R^T diag(lambda) R for symmetric masks
    x = rng.uniform(size=(n, n))
    lam_signed = oracle.tensor_apply(1, oracle.apply(p, oracle.tensor_apply(-1, np.eye(n * n)[0].reshape(n, n)),
                                                     path=1, bc=REFL))
    eig = np.empty((n, n))
    for a in range(n):
        for b in range(n):
            s1 = np.arange(-2, 3)
            eig[a, b] = sum(p[2 + i, 2 + j] * np.cos(i * a * np.pi / n) * np.cos(j * b * np.pi / n)
                            for i in s1 for j in s1)
    Ax = oracle.precondition_apply(eig, x, bc=REFL)
    assert rel(Ax, oracle.apply(p, x, path=1, bc=REFL)) <= 1e-13
    del lam_signed


def test_oracle_reflective_delta_landweber(oracle):
    # D-Landweber with a delta mask and alpha: x_1 = g / (1 + alpha) (solver_test.cpp:133-150)
    rng = np.random.default_rng(3)
    g = rng.uniform(size=(6, 6))
    delta = np.zeros((3, 3))
    delta[1, 1] = 1.0
    d = oracle.build_tikhonov(delta, 0.25, 6, 6, bc=REFL)
    run = oracle.landweber(delta, g, d=d, max_iters=1, stop=oracle.STOP_FIXED, fixed_iters=1, keep_iterates=True,
                           bc=REFL)
    assert np.abs(run["iterates"][0] - g / 1.25).max() <= 1e-14


# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("n1,n2,q1,q2", [(16, 16, 1, 2), (64, 48, 5, 7), (96, 128, 9, 12), (37, 53, 3, 5)])
def test_gpu_reflective_blur(dbx, oracle, n1, n2, q1, q2):
    rng = np.random.default_rng(n1 + q1)
    t = rand_psf(rng, q1, q2)
    f = rng.uniform(size=(n1, n2))
    op = dbx.BlurOperator(dbx.Psf(t), dbx.BoundaryCondition.Reflective, n1, n2)
    for conv in (dbx.ConvEngine.Auto, dbx.ConvEngine.Fft, dbx.ConvEngine.Direct):
        op.set_conv(conv)
        assert rel(dbx.apply(op, f), oracle.apply(t, f, bc=REFL)) <= 1e-12, conv
        assert rel(dbx.apply_reblur_adjoint(op, f), oracle.apply(t, f, adjoint=True, bc=REFL)) <= 1e-12, conv


@pytest.mark.gpu
@pytest.mark.parametrize("n1,n2", [(16, 16), (64, 48), (256, 128), (7, 9), (100, 64)])
@pytest.mark.parametrize("engine", ["Auto", "Dense"])
def test_gpu_cosine3_and_precondition(dbx, oracle, n1, n2, engine):
    """Compiled DCT lengths run the FFT form; others (7, 9, 100) the dense GEMM form."""
    rng = np.random.default_rng(n1 * 7 + n2)
    x = rng.uniform(-1, 1, (n1, n2))
    eng = getattr(dbx.DstEngine, engine)
    assert rel(dbx.tensor_apply(dbx.TransformKind.CosineIII, x, engine=eng), oracle.tensor_apply(1, x)) <= 1e-12
    t = rand_psf(rng, 2, 3)
    d = dbx.build_tikhonov(dbx.Psf(t), dbx.PreconditionerSpec(dbx.Algebra.CosineIII, 0.02), n1, n2)
    dref = oracle.build_tikhonov(t, 0.02, n1, n2, bc=REFL)
    assert rel(d.eigs, dref) <= 1e-14
    assert rel(dbx.precondition_apply(d, x, engine=eng), oracle.precondition_apply(dref, x, bc=REFL)) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("n,iters,precond", [(64, 12, True), (96, 10, True), (64, 12, False), (100, 8, True)])
def test_gpu_reflective_landweber_trajectory(dbx, oracle, n, iters, precond):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C1"]
    f, g, taps = cf.make_problem(c, n=n)
    op = dbx.BlurOperator(dbx.Psf(taps), dbx.BoundaryCondition.Reflective, n, n)
    cfg = dbx.SolverConfig(max_iters=iters, track_rre_against=f)
    if precond:
        d = dbx.build_tikhonov(dbx.Psf(taps), dbx.PreconditionerSpec(dbx.Algebra.CosineIII, c.alpha), n, n)
        run = dbx.d_landweber(op, d, g, cfg, keep_iterates=True)
        ref = oracle.landweber(taps, g, d=oracle.build_tikhonov(taps, c.alpha, n, n, bc=REFL), f_true=f,
                               max_iters=iters, keep_iterates=True, bc=REFL)
    else:
        run = dbx.landweber(op, g, cfg, keep_iterates=True)
        ref = oracle.landweber(taps, g, f_true=f, max_iters=iters, keep_iterates=True, bc=REFL)
    assert run.iterations_executed == ref["iterations_executed"]
    assert run.best_iteration == ref["best_iteration"]
    for k in range(iters):
        assert rel(run.iterates[k], ref["iterates"][k]) <= 1e-10, k + 1
    np.testing.assert_allclose(run.residual_history, ref["residual_history"], rtol=1e-10, atol=0)
    # the AR algebra is refused for reflective BCs (and vice versa)
    if precond:
        dar = dbx.build_tikhonov(dbx.Psf(taps), dbx.PreconditionerSpec(dbx.Algebra.AntiReflective, c.alpha), n, n)
        with pytest.raises(ValueError):
            dbx.d_landweber(op, dar, g, cfg)
