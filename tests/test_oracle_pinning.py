"""Pins the CPU oracle (oracle/deblur_oracle.cpp) to the reference's own test
assertions before it is trusted to certify the GPU path.  Each test re-states
one reference GoogleTest (file:line under /root/reference/proj/tests/) with an
independent numpy re-derivation as the dense oracle, as the reference does with
tests/oracle/*.hpp.  CPU only.
"""
import numpy as np
import pytest


def rand_psf(rng, q1, q2):  # tests/oracle/helpers.hpp:25-29 (uniform [0.05,1], normalised)
    t = rng.uniform(0.05, 1.0, (2 * q1 + 1, 2 * q2 + 1))
    return t / t.sum()


def sym_psf(rng, q1, q2):  # helpers.hpp:31-33
    t = rand_psf(rng, q1, q2)
    return (t + t[::-1, :] + t[:, ::-1] + t[::-1, ::-1]) / 4.0


def literal_pad(f, q1, q2):
    """AR branch of tests/oracle/helpers.hpp:82-172, 1-based index transcription."""
    n1, n2 = f.shape
    out = np.zeros((n1 + 2 * q1, n2 + 2 * q2))
    fov = lambda i1, i2: f[i1 - 1, i2 - 1]

    def put(i1, i2, v):
        out[i1 - 1 + q1, i2 - 1 + q2] = v

    for i1 in range(1, n1 + 1):
        for i2 in range(1, n2 + 1):
            put(i1, i2, fov(i1, i2))
    for i1 in range(1, n1 + 1):
        for i2 in range(1, q2 + 1):
            put(i1, 1 - i2, 2 * fov(i1, 1) - fov(i1, i2 + 1))
            put(i1, n2 + i2, 2 * fov(i1, n2) - fov(i1, n2 - i2))
    for i1 in range(1, q1 + 1):
        for i2 in range(1, n2 + 1):
            put(1 - i1, i2, 2 * fov(1, i2) - fov(i1 + 1, i2))
            put(n1 + i1, i2, 2 * fov(n1, i2) - fov(n1 - i1, i2))
    for i1 in range(1, q1 + 1):
        for i2 in range(1, q2 + 1):
            put(1 - i1, 1 - i2, 4 * fov(1, 1) - 2 * fov(1, i2 + 1) - 2 * fov(i1 + 1, 1) + fov(i1 + 1, i2 + 1))
            put(1 - i1, n2 + i2, 4 * fov(1, n2) - 2 * fov(1, n2 - i2) - 2 * fov(i1 + 1, n2) + fov(i1 + 1, n2 - i2))
            put(n1 + i1, 1 - i2, 4 * fov(n1, 1) - 2 * fov(n1, i2 + 1) - 2 * fov(n1 - i1, 1) + fov(n1 - i1, i2 + 1))
            put(n1 + i1, n2 + i2,
                4 * fov(n1, n2) - 2 * fov(n1, n2 - i2) - 2 * fov(n1 - i1, n2) + fov(n1 - i1, n2 - i2))
    return out


def numpy_apply(t, f):
    """Independent A f: literal pad + explicit valid correlation (blur.hpp:39-52)."""
    q1, q2 = (t.shape[0] - 1) // 2, (t.shape[1] - 1) // 2
    P = literal_pad(f, q1, q2)
    n1, n2 = f.shape
    g = np.zeros((n1, n2))
    for s1 in range(-q1, q1 + 1):
        for s2 in range(-q2, q2 + 1):
            g += t[q1 + s1, q2 + s2] * P[q1 - s1:q1 - s1 + n1, q2 - s2:q2 - s2 + n2]
    return g


def dense_op(fn, n1, n2):
    A = np.zeros((n1 * n2, n1 * n2))
    for j in range(n1 * n2):
        e = np.zeros(n1 * n2)
        e[j] = 1.0
        A[:, j] = fn(e.reshape(n1, n2)).ravel()
    return A


def dense_sine1(m):  # dense_transforms.hpp:34-41 (integer-reduced argument)
    s = np.arange(1, m + 1)
    e = np.outer(s, s) % (2 * (m + 1))
    return np.sqrt(2.0 / (m + 1)) * np.sin(np.pi * e / (m + 1))


def ar_params(m):
    p = 1.0 - np.arange(1, m - 1) / (m - 1)
    return p, np.sqrt(1.0 + p @ p)


def dense_ar_forward(m):  # dense_transforms.hpp:45-57
    p, a = ar_params(m)
    T = np.zeros((m, m))
    T[0, 0] = T[-1, -1] = 1 / a
    T[1:-1, 1:-1] = dense_sine1(m - 2)
    T[1:-1, 0] = p / a
    T[1:-1, -1] = p[::-1] / a
    return T


def dense_ar_inverse(m):  # dense_transforms.hpp:61-75
    p, a = ar_params(m)
    Q = dense_sine1(m - 2)
    T = np.zeros((m, m))
    T[0, 0] = T[-1, -1] = a
    T[1:-1, 1:-1] = Q
    T[1:-1, 0] = -(Q @ p)
    T[1:-1, -1] = -(Q @ p[::-1])
    return T


# --------------------------- boundary_test.cpp ----------------------------
def test_ar_pad_continues_ramps(oracle):  # boundary_test.cpp:28-34
    f = np.arange(1, 9, dtype=float)[None, :]
    p = oracle.pad_ar(f, 0, 3)
    assert np.abs(p[0] - (np.arange(p.shape[1]) - 2.0)).max() <= 1e-15


def test_pad_matches_literal_transcription(oracle):  # boundary_test.cpp:36-45
    rng = np.random.default_rng(31)
    f = rng.uniform(0, 1, (6, 7))
    assert np.abs(oracle.pad_ar(f, 2, 3) - literal_pad(f, 2, 3)).max() <= 1e-14


def test_support_condition(oracle):  # boundary_test.cpp:47-56
    with pytest.raises(ValueError):
        oracle.pad_ar(np.ones((4, 4)), 3, 0)
    oracle.pad_ar(np.ones((4, 4)), 2, 2)
    oracle.pad_ar(np.ones((1, 9)), 0, 3)


# ------------------------------ blur_test.cpp -----------------------------
def test_delta_and_constant(oracle):  # blur_test.cpp:12-31
    rng = np.random.default_rng(41)
    f = rng.uniform(0, 1, (6, 5))
    d = np.zeros((3, 3))
    d[1, 1] = 1
    assert np.abs(oracle.apply(d, f) - f).max() <= 1e-15
    t = rand_psf(rng, 2, 1)
    c = np.full((7, 7), 4.5)
    assert np.abs(oracle.apply(t, c) - c).max() <= 1e-13


def test_apply_matches_dense(oracle):  # blur_test.cpp:33-44
    rng = np.random.default_rng(47)
    t = rand_psf(rng, 1, 2)
    f = rng.uniform(0, 1, (7, 8))
    A = dense_op(lambda e: numpy_apply(t, e), 7, 8)
    want = A @ f.ravel()
    got = oracle.apply(t, f).ravel()
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12


def test_fft_path_agrees_with_direct(oracle):  # blur_test.cpp:46-59
    rng = np.random.default_rng(53)
    t = rand_psf(rng, 1, 9)
    f = rng.uniform(0, 1, (24, 30))
    direct = oracle.apply(t, f, path=1)
    fast = oracle.apply(t, f, path=2)
    assert np.abs(fast - direct).max() <= 1e-12
    assert np.abs(oracle.apply(t, f) - fast).max() <= 1e-12  # auto picks FFT for q > 7


def test_reblur_is_rotated_operator(oracle):  # blur_test.cpp:80-105
    rng = np.random.default_rng(61)
    ts = sym_psf(rng, 1, 1)
    r = rng.uniform(0, 1, (6, 6))
    assert np.abs(oracle.apply(ts, r, adjoint=True) - oracle.apply(ts, r)).max() <= 1e-15
    t = rand_psf(rng, 2, 1)
    assert np.abs(oracle.apply(t, r, adjoint=True) - numpy_apply(t[::-1, ::-1], r)).max() <= 1e-14


def test_1d_ar_structure(oracle):  # blur_test.cpp:116-139 (Eq. ARnosym1D)
    rng = np.random.default_rng(71)
    n, q = 7, 3
    t = rand_psf(rng, 0, q)
    A = dense_op(lambda e: oracle.apply(t, e), 1, n)
    h = lambda k: t[0, q + k]
    for k in range(q + 1):
        v = h(k) + 2 * sum(h(j) for j in range(k + 1, q + 1))
        w = h(-k) + 2 * sum(h(-j) for j in range(k + 1, q + 1))
        assert abs(A[k, 0] - v) <= 1e-15 and abs(A[n - 1 - k, n - 1] - w) <= 1e-15
    for k in range(1, n - 1):
        u = h(-k) - h(k) if k <= q else 0.0
        assert abs(A[0, k] - u) <= 1e-15 and abs(A[n - 1, n - 1 - k] + u) <= 1e-15
    assert A[0, n - 1] == 0.0 and A[n - 1, 0] == 0.0


# --------------------------- transforms_test.cpp --------------------------
def test_sine1_involutory_and_dense(oracle):  # transforms_test.cpp:43-58, 138-164
    rng = np.random.default_rng(103)
    v = rng.uniform(-1, 1, 15)
    assert np.abs(oracle.sine1_forward(oracle.sine1_forward(v)) - v).max() <= 1e-13
    assert abs(oracle.sine1_forward(np.array([-3.0]))[0] + 3.0) <= 1e-15
    for m in range(2, 65):
        Q = dense_sine1(m)
        QQ = np.stack([oracle.sine1_forward(oracle.sine1_forward(np.eye(m)[j])) for j in range(m)], 1)
        assert np.abs(QQ - np.eye(m)).max() <= 1e-12, m
        x = rng.uniform(-1, 1, m)
        assert np.abs(oracle.sine1_forward(x) - Q @ x).max() <= 1e-12, m


def test_ar_transform_known_answers(oracle):  # transforms_test.cpp:60-90, 120-130
    a, p = oracle.make_ar_transform(5)
    assert np.allclose(p, [0.75, 0.5, 0.25], atol=1e-15, rtol=0)
    w = oracle.ar_forward(np.eye(5)[0])
    assert np.abs(w - np.array([1, 0.75, 0.5, 0.25, 0]) / a).max() <= 1e-14
    rng = np.random.default_rng(109)
    v = rng.uniform(-1, 1, 9)
    v[0] = v[-1] = 0.0
    w = oracle.ar_forward(v)
    assert w[0] == 0.0 and w[-1] == 0.0
    assert np.abs(w[1:-1] - oracle.sine1_forward(v[1:-1])).max() <= 1e-14
    a6, p6 = oracle.make_ar_transform(6)
    u = oracle.ar_inverse(np.eye(6)[0])
    assert abs(u[0] - a6) <= 1e-14 and abs(u[-1]) <= 1e-14
    assert np.abs(u[1:-1] + oracle.sine1_forward(p6)).max() <= 1e-13


def test_ar_transform_dense_and_inverse(oracle):  # transforms_test.cpp:92-118, 154-172
    rng = np.random.default_rng(113)
    for m in range(3, 65):
        v = rng.uniform(-1, 1, m)
        assert np.abs(oracle.ar_forward(v) - dense_ar_forward(m) @ v).max() <= 1e-12, m
        assert np.abs(oracle.ar_inverse(v) - dense_ar_inverse(m) @ v).max() <= 1e-12, m
        assert np.abs(oracle.ar_forward(oracle.ar_inverse(v)) - v).max() <= 1e-12, m
        T = dense_ar_forward(m)
        assert abs(np.linalg.norm(T[:, 0]) - 1) <= 1e-14 and abs(np.linalg.norm(T[:, -1]) - 1) <= 1e-14
    with pytest.raises(ValueError):
        oracle.make_ar_transform(2)


def test_tensor_apply_kronecker(oracle):  # transforms_test.cpp:184-213
    rng = np.random.default_rng(139)
    n1, n2 = 8, 10
    x = rng.uniform(-1, 1, (n1, n2))
    for kind, k1, k2 in ((oracle.KIND_SINEI, dense_sine1(n1), dense_sine1(n2)),
                         (oracle.KIND_AR, dense_ar_forward(n1), dense_ar_forward(n2)),
                         (oracle.KIND_ARINV, dense_ar_inverse(n1), dense_ar_inverse(n2))):
        want = np.kron(k1, k2) @ x.ravel()
        assert np.abs(oracle.tensor_apply(kind, x).ravel() - want).max() <= 1e-12


# ---------------------------- spectral_test.cpp ---------------------------
def test_ar_eigenvalues(oracle):  # spectral_test.cpp:90-120
    rng = np.random.default_rng(179)
    p = sym_psf(rng, 1, 1)
    e = oracle.eig_antireflective(p, 7, 8)
    for v in (e[0, 0], e[0, 7], e[6, 0], e[6, 7]):
        assert abs(v - 1.0) <= 1e-14
    assert np.array_equal(e[0], e[6]) and np.array_equal(e[:, 0], e[:, 7])
    d = np.zeros((3, 3))
    d[1, 1] = 1
    assert np.abs(oracle.eig_antireflective(d, 6, 6) - 1).max() <= 1e-15
    A = dense_op(lambda x: numpy_apply(p, x), 7, 8)
    dense = np.sort(np.linalg.eigvals(A).real)
    assert np.abs(np.sort(e.ravel()) - dense).max() <= 1e-8
    assert int(np.sum(np.abs(e.ravel() - 1.0) <= 1e-12)) == 4
    with pytest.raises(ValueError):
        oracle.eig_antireflective(rand_psf(rng, 1, 1), 7, 8)


def test_filter_apply_reconstructs_blur(oracle):  # spectral_test.cpp:151-186
    rng = np.random.default_rng(197)
    for _ in range(3):
        p = sym_psf(rng, 2, 1)
        v = rng.uniform(-1, 1, (16, 16))
        lam = oracle.eig_antireflective(p, 16, 16)
        via_filter = oracle.precondition_apply(lam, v)
        assert np.linalg.norm(via_filter - oracle.apply(p, v)) <= 1e-10 * np.linalg.norm(v)


def test_theorem1_reconstruction(oracle):  # oracles_test.cpp:102-115
    rng = np.random.default_rng(233)
    p = sym_psf(rng, 1, 1)
    n1, n2 = 7, 8
    A = dense_op(lambda x: numpy_apply(p, x), n1, n2)
    lam = oracle.eig_antireflective(p, n1, n2).ravel()
    T = np.kron(dense_ar_forward(n1), dense_ar_forward(n2))
    Tt = np.kron(dense_ar_inverse(n1), dense_ar_inverse(n2))
    assert np.abs(T @ np.diag(lam) @ Tt - A).max() <= 1e-10


# ------------------------- preconditioner_test.cpp ------------------------
def test_tikhonov_values(oracle):  # preconditioner_test.cpp:67-113
    d = np.zeros((3, 3))
    d[1, 1] = 1
    assert np.abs(oracle.build_tikhonov(d, 0.0, 6, 6) - 1).max() <= 1e-15
    base = np.array([[0.0, 0.5]])
    assert abs(oracle.tikhonov_filter(base, 0.1)[0, 0] - 10.0) <= 1e-15
    with pytest.raises(ValueError):
        oracle.tikhonov_filter(base, 0.0)
    rng = np.random.default_rng(313)
    t = rand_psf(rng, 2, 2)
    dd = oracle.build_tikhonov(t, 0.05, 9, 9)
    assert dd.min() > 0 and dd.max() <= 1 / 0.05 + 1e-15
    lam = np.abs(oracle.eig_antireflective(oracle.symmetrize(t), 9, 9).ravel())
    o = np.argsort(lam)
    assert np.all(np.diff(dd.ravel()[o])[np.diff(lam[o]) > 1e-12] < 0)


def test_precondition_apply_dense(oracle):  # preconditioner_test.cpp:125-150
    rng = np.random.default_rng(337)
    p = sym_psf(rng, 1, 1)
    n1, n2 = 6, 7
    d = oracle.build_tikhonov(p, 0.02, n1, n2)
    r = rng.uniform(0, 1, (n1, n2))
    T = np.kron(dense_ar_forward(n1), dense_ar_forward(n2))
    Tt = np.kron(dense_ar_inverse(n1), dense_ar_inverse(n2))
    want = T @ np.diag(d.ravel()) @ Tt @ r.ravel()
    assert np.abs(oracle.precondition_apply(d, r).ravel() - want).max() <= 1e-11
    huge = oracle.build_tikhonov(rand_psf(rng, 1, 1), 1e12, 8, 8)
    r8 = rng.uniform(0, 1, (8, 8))
    assert np.linalg.norm(oracle.precondition_apply(huge, r8)) <= 1e-10 * np.linalg.norm(r8)


# ------------------------------ image_test.cpp ----------------------------
def test_noise_exact_level_and_determinism(oracle):  # image_test.cpp:12-34
    rng = np.random.default_rng(5)
    g = rng.uniform(10, 200, (12, 9))
    out = oracle.add_noise(g, 0.001, 99)
    assert abs(np.linalg.norm(out - g) / np.linalg.norm(g) - 0.001) <= 1e-12
    assert np.array_equal(oracle.add_noise(g, 0.01, 4242), oracle.add_noise(g, 0.01, 4242))
    assert not np.array_equal(oracle.add_noise(g, 0.01, 4242), oracle.add_noise(g, 0.01, 4243))
    assert np.array_equal(oracle.add_noise(g, 0.0, 1), g)


# ------------------------------ solver_test.cpp ---------------------------
def test_dlandweber_delta_mask(oracle):  # solver_test.cpp:133-150
    rng = np.random.default_rng(397)
    g = rng.uniform(1, 2, (8, 8))
    d = np.zeros((1, 1))
    d[0, 0] = 1.0
    for alpha, want in ((0.25, g / 1.25), (0.0, g)):
        D = oracle.build_tikhonov(d, alpha, 8, 8)
        run = oracle.landweber(d, g, d=D, stop=oracle.STOP_FIXED, fixed_iters=1, max_iters=1)
        assert np.abs(run["restored"] - want).max() <= 1e-12


def test_identity_filter_is_plain(oracle):  # solver_test.cpp:111-131 (AR variant)
    rng = np.random.default_rng(389)
    t = rand_psf(rng, 1, 1)
    f = rng.uniform(1, 2, (12, 12))
    g = oracle.add_noise(oracle.apply(t, f), 0.001, 7)
    a = oracle.landweber(t, g, f_true=f, stop=oracle.STOP_FIXED, fixed_iters=100)
    b = oracle.landweber(t, g, d=np.ones((12, 12)), f_true=f, stop=oracle.STOP_FIXED, fixed_iters=100)
    assert np.abs(a["rre_history"] - b["rre_history"]).max() <= 1e-12
    assert np.abs(a["restored"] - b["restored"]).max() <= 1e-12


def test_guard_zero_iters_and_residual_rule(oracle):  # solver_test.cpp:27-39, 85-109
    rng = np.random.default_rng(379)
    f = rng.uniform(1, 2, (8, 8))
    d = np.zeros((3, 3))
    d[1, 1] = 1
    with pytest.raises(oracle.OracleDivergence):
        oracle.landweber(d, f, tau=3.0, stop=oracle.STOP_FIXED, fixed_iters=200, max_iters=200)
    z = oracle.landweber(d, f, f_true=f, stop=oracle.STOP_FIXED, fixed_iters=0)
    assert z["iterations_executed"] == 0 and np.abs(z["restored"]).max() == 0.0
    t = 0.4 * sym_psf(rng, 1, 1)
    t[1, 1] += 0.6  # well-conditioned AR operator (the reference uses Reflective BCs here)
    f10 = rng.uniform(1, 2, (10, 10))
    g = oracle.apply(t, f10)
    run = oracle.landweber(t, g, max_iters=500, stop=oracle.STOP_RESID, resid_eps=1e-3)
    assert run["iterations_executed"] < 500
    assert run["residual_history"][-1] / np.linalg.norm(g) < 1e-3


def test_histories_deterministic(oracle):  # solver_test.cpp:257-274
    rng = np.random.default_rng(401)
    t = rand_psf(rng, 1, 1)
    f = rng.uniform(1, 2, (10, 10))
    g = oracle.add_noise(oracle.apply(t, f), 0.001, 31337)
    a = oracle.landweber(t, g, f_true=f, max_iters=50)
    b = oracle.landweber(t, g, f_true=f, max_iters=50)
    assert np.array_equal(a["rre_history"], b["rre_history"])
    assert np.array_equal(a["residual_history"], b["residual_history"])


def _ref_scene(n, pad):  # synthetic.hpp:15-40
    r = (np.arange(n + 2 * pad) - pad + 0.5) / n
    u, v = np.meshgrid(r, r, indexing="ij")
    s = 40.0 + 110.0 * u + 55.0 * v
    s += 62.0 * (((u - 0.34) ** 2 + (v - 0.38) ** 2) < 0.17 ** 2)
    s += 48.0 * ((u > 0.56) & (u < 0.82) & (v > 0.14) & (v < 0.42))
    s += 36.0 * np.exp(-((u - 0.70) ** 2 + (v - 0.76) ** 2) / (2 * 0.11 ** 2))
    return s


def _ref_gaussian_portion(sigma, q1, q2, o1, o2):  # psf.hpp:126-138
    i1 = np.arange(-q1, q1 + 1)[:, None] - o1
    i2 = np.arange(-q2, q2 + 1)[None, :] - o2
    t = np.exp(-(i1 * i1 + i2 * i2) / (2 * sigma * sigma))
    return t / t.sum()


@pytest.mark.slow
def test_acceleration_trend(oracle):  # solver_test.cpp:164-210 (AR branch)
    n = 64
    p = _ref_gaussian_portion(1.6, 5, 5, 0.3, 0.15)
    scene = _ref_scene(n, 5)
    f = scene[5:5 + n, 5:5 + n]
    g = np.zeros((n, n))
    for s1 in range(-5, 6):
        for s2 in range(-5, 6):
            g += p[5 + s1, 5 + s2] * scene[5 - s1:5 - s1 + n, 5 - s2:5 - s2 + n]
    g = oracle.add_noise(g, 0.001, 2024)
    plain = oracle.landweber(p, g, f_true=f, max_iters=1500)
    target = 1.01 * plain["rre_history"][plain["best_iteration"] - 1]
    first = 0
    for alpha in (1e-3, 1e-2, 1e-1):
        D = oracle.build_tikhonov(p, alpha, n, n)
        fast = oracle.landweber(p, g, d=D, f_true=f, max_iters=200)
        hit = np.nonzero(fast["rre_history"] <= target)[0]
        if len(hit):
            first = hit[0] + 1 if first == 0 else min(first, hit[0] + 1)
    assert first > 0
    assert plain["best_iteration"] >= 5 * first


# ---------------------------------------------------------------------------
# Oracle engineering: the Stockham/Bluestein FFT, line-parallel threads and
# the kernel-spectrum cache must not change any number; the long-double
# variant is the same algorithm with a 64-bit mantissa.
@pytest.mark.parametrize("n", [1, 2, 3, 4, 5, 7, 12, 31, 62, 97, 255, 271, 1023, 1084, 2172, 4096])
def test_fft_against_numpy(oracle, n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    for sign in (-1, 1):
        got = oracle.fft(x, sign)
        want = np.fft.fft(x) if sign < 0 else np.fft.ifft(x) * n
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-14


def test_oracle_threads_and_kernel_cache_bit_identical(oracle):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C3"]
    f, g, taps = cf.make_problem(c, n=72)
    d = oracle.build_tikhonov(taps, c.alpha, 72, 72)
    runs = []
    try:
        for threads, cache in ((1, False), (5, False), (3, True)):
            oracle.set_threads(threads)
            oracle.set_kernel_cache(cache)
            runs.append(oracle.landweber(taps, g, d=d, f_true=f, max_iters=6, keep_iterates=True))
    finally:
        oracle.set_threads(1)
        oracle.set_kernel_cache(False)
    for r in runs[1:]:
        assert np.array_equal(r["iterates"], runs[0]["iterates"])
        assert np.array_equal(r["rre_history"], runs[0]["rre_history"])


def test_long_double_oracle_is_the_same_algorithm(oracle):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C2"]
    n = 48
    f, g, taps = cf.make_problem(c, n=n)
    dbl = oracle.landweber(taps, g, d=oracle.build_tikhonov(taps, c.alpha, n, n), f_true=f, max_iters=8,
                           keep_iterates=True)
    ld = oracle.landweber(taps, g, f_true=f, max_iters=8, keep_iterates=True, long_double_alpha=c.alpha)
    for k in range(8):
        e = np.linalg.norm(dbl["iterates"][k] - ld["iterates"][k]) / np.linalg.norm(ld["iterates"][k])
        assert 0 < e <= 1e-13
    assert dbl["best_iteration"] == ld["best_iteration"]
    x = np.random.default_rng(3).standard_normal((n, n))
    for kind in (3, 4):
        a, b = oracle.tensor_apply(kind, x), oracle.tensor_apply(kind, x, long_double=True)
        assert 0 < np.linalg.norm(a - b) / np.linalg.norm(b) <= 1e-14
