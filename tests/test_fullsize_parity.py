"""Full-size, every-iteration parity of the production GPU path against the
CPU oracle on all five BASELINE configs (north_star: relative L2 <= 1e-10 at
EVERY iteration, identical best-RRE iteration; solver.hpp:101-131, strict
'<' at :114).

* C1 256^2 x 50 (tests/test_gpu_parity.py covers it at full length already)
* C2 512^2 x 100, plain and D-Landweber
* C3 the benchmarked batch: 64 x 1024^2 x 40 in ONE batch run (the bench's
  plan and pipeline), images 0 / 21 / 42 / 63 taken from that run
* C4 2048^2 x 30
* C5 8192^2 x 5 through the single-image path, and through the row-slab
  decomposition at P = 2 (two simulated ranks in one process)

The oracle runs line-parallel on every host core with the mask spectrum
kept between calls (both change no number: tests/test_oracle_pinning.py
checks bit-identity), so the whole module takes a few minutes.  The FP64
rounding floor of both sides against a long-double oracle and the best vs
runner-up RRE margins are reported by tools/parity_report.py
(profiles/r02_parity_report.json).
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ITER_TOL = 1e-10
HIST_RTOL = 1e-10


def rel(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


@pytest.fixture(scope="module")
def dev(dbx):
    if dbx.lib().dbx_device_count() < 1:
        pytest.fail("no sm_100 device visible: GPU tests must run on a B200")
    return dbx


@pytest.fixture(scope="module")
def orc(oracle):
    oracle.set_threads(os.cpu_count() or 1)
    oracle.set_kernel_cache(True)
    yield oracle
    oracle.set_kernel_cache(False)
    oracle.set_threads(1)


def check_run(iters_gpu, rre_gpu, res_gpu, best_gpu, done_gpu, ref, label):
    """iters_gpu: callable k -> x_k (numpy) for k = 1..done."""
    assert done_gpu == ref["iterations_executed"], label
    assert best_gpu == ref["best_iteration"], label
    np.testing.assert_allclose(res_gpu, ref["residual_history"], rtol=HIST_RTOL, atol=0, err_msg=label)
    if len(ref["rre_history"]):
        np.testing.assert_allclose(rre_gpu, ref["rre_history"], rtol=HIST_RTOL, atol=0, err_msg=label)
    worst = 0.0
    for k in range(1, done_gpu + 1):
        e = rel(iters_gpu(k), ref["iterates"][k - 1])
        worst = max(worst, e)
        assert e <= ITER_TOL, (label, k, e)
    return worst


def _single(dev, orc, name, iters=None, precond=True, problem=None, ref=None):
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS[name]
    n = c.n
    iters = iters or c.iters
    f, g, taps = problem or cf.make_problem(c)
    op = dev.BlurOperator(dev.Psf(taps), dev.BoundaryCondition.AntiReflective, n, n)
    cfg = dev.SolverConfig(max_iters=iters, track_rre_against=f)
    if precond:
        d = dev.build_tikhonov(dev.Psf(taps), dev.PreconditionerSpec(dev.Algebra.AntiReflective, c.alpha), n, n)
        run = dev.d_landweber(op, d, g, cfg, keep_iterates=True)
        if ref is None:
            ref = orc.landweber(taps, g, d=orc.build_tikhonov(taps, c.alpha, n, n), f_true=f, max_iters=iters,
                                keep_iterates=True)
    else:
        run = dev.landweber(op, g, cfg, keep_iterates=True)
        ref = orc.landweber(taps, g, f_true=f, max_iters=iters, keep_iterates=True)
    check_run(lambda k: run.iterates[k - 1], run.rre_history, run.residual_history, run.best_iteration,
              run.iterations_executed, ref, f"{name} precond={precond}")
    assert rel(run.restored, ref["restored"]) <= ITER_TOL
    return op


@pytest.mark.parametrize("precond", [False, True])
def test_c2_full_size_100_iterations(dev, orc, precond):
    _single(dev, orc, "C2", precond=precond)


def test_c4_full_size_30_iterations(dev, orc):
    _single(dev, orc, "C4")


C5_ITERS = 5


@pytest.fixture(scope="module")
def c5(orc):
    """C5 problem and its oracle trajectory (shared by the two C5 tests)."""
    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C5"]
    f, g, taps = cf.make_problem(c)
    ref = orc.landweber(taps, g, d=orc.build_tikhonov(taps, c.alpha, c.n, c.n), f_true=f, max_iters=C5_ITERS,
                        keep_iterates=True)
    return (f, g, taps), ref


def test_c5_full_size_single_image(dev, orc, c5):
    _single(dev, orc, "C5", iters=C5_ITERS, problem=c5[0], ref=c5[1])


def test_c3_benchmarked_batch_every_iteration(dev, orc):
    """The bench's C3 config: one 64-image plan (fused separable pipeline,
    CUDA graph) with every iterate kept on the device; four images of that
    batch run against the oracle for all 40 iterations."""
    import ctypes as C

    import torch

    from paper_1211_0393_b200 import configs as cf
    c = cf.CONFIGS["C3"]
    n, q, H, B = c.n, c.q, c.iters, c.batch
    N = n * n
    L = dev.lib()
    F, G, taps = cf.make_batch(c, B)
    d0 = torch.device("cuda", 0)
    g = torch.from_numpy(G).to(d0)
    f = torch.from_numpy(F).to(d0)
    out = torch.empty_like(g)
    xh = torch.empty((B, H, n, n), dtype=torch.float64, device=d0)
    plan = C.c_void_p()
    dev._check(L.dbx_plan_create(n, n, B, dev._ptr(taps), q, q, 3, 0, C.byref(plan)))
    try:
        dev._check(L.dbx_precond_build(plan, float(c.alpha)))
        rre = np.zeros((B, H))
        res = np.zeros((B, H))
        best, done = (C.c_int * B)(), (C.c_int * B)()
        dev._check(L.dbx_landweber_run(plan, dev._ptr(g), dev._ptr(f), 1.0, H, 1, 0, 0.0, 1, dev._ptr(out),
                                       dev._ptr(rre), dev._ptr(res), best, done, dev._ptr(xh)))
        fz = C.c_int()
        L.dbx_plan_pipeline(plan, C.byref(fz))
        assert fz.value == 2, "C3 must run the fused separable pipeline (the benchmarked one)"
    finally:
        L.dbx_plan_destroy(plan)
    del g, out
    dref = orc.build_tikhonov(taps, c.alpha, n, n)
    for b in (0, 21, 42, 63):
        ref = orc.landweber(taps, G[b], d=dref, f_true=F[b], max_iters=H, keep_iterates=True)
        xb = xh[b].cpu().numpy()
        check_run(lambda k: xb[k - 1], rre[b], res[b], best[b], done[b], ref, f"C3 image {b}")


def test_c5_row_slabs_p2_every_iteration(dev, orc, c5):
    """C5 8192^2 through the row-slab decomposition (2 simulated ranks:
    halo exchange for the blur, all-to-all transposes for the column DSTs)
    against the oracle at every iteration."""
    import torch

    from paper_1211_0393_b200 import configs as cf
    from paper_1211_0393_b200.slab import LocalWorld, SlabLandweber
    c = cf.CONFIGS["C5"]
    n, iters, P = c.n, C5_ITERS, 2
    (f, g, taps), ref = c5
    R = n // P
    d0 = torch.device("cuda", 0)
    gs = {p: torch.from_numpy(np.ascontiguousarray(g[p * R:(p + 1) * R])).to(d0) for p in range(P)}
    fs = {p: torch.from_numpy(np.ascontiguousarray(f[p * R:(p + 1) * R])).to(d0) for p in range(P)}
    xs = {}

    def keep(k, slabs):
        xs[k] = np.concatenate([slabs[p].cpu().numpy() for p in range(P)])

    solver = SlabLandweber(LocalWorld(P), n, taps, c.q, c.alpha, device=0)
    try:
        run = solver.run(gs, fs, iters, on_iterate=keep)
    finally:
        solver.close()
    check_run(lambda k: xs[k], run["rre_history"], run["residual_history"], run["best_iteration"],
              run["iterations_executed"], ref, "C5 slabs P=2")


@pytest.mark.parametrize("P", [1, 2])
def test_c5_cpp_slab_loop_every_iteration(dev, orc, c5, P):
    """C5 8192^2 through the C++ row-slab loop (dbx_slab_run: separable direct
    blur on halo-extended slabs, fused T~ d^T T column blocks, device-side
    norms and bookkeeping) with P in-process ranks, against the oracle at every
    iteration."""
    import torch

    from paper_1211_0393_b200 import configs as cf
    from paper_1211_0393_b200.slab import SlabRun
    c = cf.CONFIGS["C5"]
    n, iters = c.n, C5_ITERS
    (f, g, taps), ref = c5
    d0 = torch.device("cuda", 0)
    gt, ft = torch.from_numpy(g).to(d0), torch.from_numpy(f).to(d0)
    run = SlabRun(n, P, taps, c.q, c.alpha, rank=-1, device=0)
    try:
        assert run.separable and run.local_slabs == P
        out, h = run.run(gt, ft, iters, keep_iterates=True)
        xs = h["iterates"]
        check_run(lambda k: xs[k - 1].cpu().numpy(), h["rre_history"], h["residual_history"], h["best_iteration"],
                  h["iterations_executed"], ref, f"C5 C++ slabs P={P}")
        best = h["best_iteration"]
        assert rel(out.cpu().numpy(), ref["iterates"][best - 1]) <= ITER_TOL
    finally:
        run.close()
