"""Row-slab decomposition of one image: the exchange layer
over gloo (world size 2, CPU) against the in-process LocalWorld, and — on the
GPU — the slab D-Landweber (P simulated ranks in one process) against the
single-image path, which tests/test_gpu_parity.py pins to the oracle."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

from paper_1211_0393_b200.slab import LocalWorld, slab_rows_of


def test_slab_rows_validation():
    assert slab_rows_of(8192, 8, 15) == 1024
    with pytest.raises(ValueError):
        slab_rows_of(100, 3, 2)
    with pytest.raises(ValueError):
        slab_rows_of(64, 8, 8)  # 8 rows < q + 1


def _local_reference(P, n, q, seed):
    rng = np.random.default_rng(seed)
    slabs = {p: torch.from_numpy(rng.uniform(size=(n // P, n))) for p in range(P)}
    w = LocalWorld(P)
    tops, bots = w.halo({p: s[:q].contiguous() for p, s in slabs.items()},
                        {p: s[-q:].contiguous() for p, s in slabs.items()})
    sends = {p: torch.from_numpy(rng.uniform(size=n * n // P)) for p in range(P)}
    recvs = {p: torch.zeros(n * n // P, dtype=torch.float64) for p in range(P)}
    w.alltoall(sends, recvs)
    return slabs, tops, bots, sends, recvs


def test_local_world_exchanges():
    P, n, q = 4, 16, 2
    slabs, tops, bots, sends, recvs = _local_reference(P, n, q, 1)
    full = torch.cat([slabs[p] for p in range(P)])
    R = n // P
    for p in range(P):
        if p > 0:
            assert torch.equal(tops[p], full[p * R - q:p * R])
        else:
            assert tops[p] is None
        if p + 1 < P:
            assert torch.equal(bots[p], full[(p + 1) * R:(p + 1) * R + q])
        else:
            assert bots[p] is None
    c = n * n // P // P
    for p in range(P):
        for s in range(P):
            assert torch.equal(recvs[s][p * c:(p + 1) * c], sends[p][s * c:(s + 1) * c])


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_1211_0393_b200.slab import DistWorld
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = 12
    slabs, tops, bots, sends, recvs = _local_reference(world, n, q, 7)
    w = DistWorld()
    t, b = w.halo({rank: slabs[rank][:q].contiguous()}, {rank: slabs[rank][-q:].contiguous()})
    assert (t[rank] is None) == (tops[rank] is None) and (b[rank] is None) == (bots[rank] is None)
    if t[rank] is not None:
        assert torch.equal(t[rank], tops[rank])
    if b[rank] is not None:
        assert torch.equal(b[rank], bots[rank])
    out = {rank: torch.zeros_like(recvs[rank])}
    w.alltoall({rank: sends[rank]}, out)
    assert torch.equal(out[rank], recvs[rank])
    tot = w.allreduce({rank: [float(rank + 1), 2.0]})
    assert tot == [float(world * (world + 1) // 2), 2.0 * world]
    dist.destroy_process_group()


def test_dist_world_matches_local_gloo():
    world = 2
    mp.spawn(_worker, args=(world, _free_port(), 2), nprocs=world, join=True)


# ---------------------------------------------------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("P,n,iters", [(1, 256, 6), (2, 256, 6), (4, 256, 6), (2, 8192, 3)])
def test_slab_landweber_matches_single_image(dbx, P, n, iters):
    """Scaled C5 problem (mask, shapes, noise, alpha) at 256^2 with 1/2/4
    simulated ranks, and the full 8192^2 FOV with 2 (Rader DSTs, conv 8640)."""
    from paper_1211_0393_b200 import configs as cf
    from paper_1211_0393_b200.slab import SlabLandweber
    c = cf.CONFIGS["C5"]
    f, g, taps = cf.make_problem(c, n=n)
    op = dbx.BlurOperator(dbx.Psf(taps), dbx.BoundaryCondition.AntiReflective, n, n)
    d = dbx.build_tikhonov(dbx.Psf(taps), dbx.PreconditionerSpec(dbx.Algebra.AntiReflective, c.alpha), n, n)
    ref = dbx.d_landweber(op, d, g, dbx.SolverConfig(max_iters=iters, track_rre_against=f))
    R = n // P
    dev = torch.device("cuda", 0)
    gs = {p: torch.from_numpy(np.ascontiguousarray(g[p * R:(p + 1) * R])).to(dev) for p in range(P)}
    fs = {p: torch.from_numpy(np.ascontiguousarray(f[p * R:(p + 1) * R])).to(dev) for p in range(P)}
    solver = SlabLandweber(LocalWorld(P), n, taps, c.q, c.alpha, device=0)
    try:
        run = solver.run(gs, fs, iters)
    finally:
        solver.close()
    assert run["iterations_executed"] == ref.iterations_executed
    assert run["best_iteration"] == ref.best_iteration
    np.testing.assert_allclose(run["residual_history"], ref.residual_history, rtol=1e-10, atol=0)
    np.testing.assert_allclose(run["rre_history"], ref.rre_history, rtol=1e-10, atol=0)
    restored = np.concatenate([run["restored"][p].cpu().numpy() for p in range(P)])
    assert np.linalg.norm(restored - ref.restored) / np.linalg.norm(ref.restored) <= 1e-10


# ---------------------------------------------------------------------------
# The C++ row-slab loop (dbx_slab_run) against the oracle
@pytest.fixture(scope="module")
def _orc_threads(oracle):
    oracle.set_threads(os.cpu_count() or 1)
    yield oracle
    oracle.set_threads(1)


@pytest.mark.gpu
@pytest.mark.parametrize("cfg,P,n,iters", [("C5", 1, 256, 8), ("C5", 2, 256, 8), ("C5", 4, 256, 8),
                                           ("C2", 2, 128, 6), ("C4", 4, 256, 4)])
def test_cpp_slab_loop_matches_oracle(dbx, _orc_threads, cfg, P, n, iters):
    """Every iterate of the C++ slab loop (P in-process ranks) vs the oracle's
    single-image run; C2 (motion mask, q = 10) and C4 (rotated Gaussian,
    q = 31) are not rank 1 and take the FFT slab blur."""
    from paper_1211_0393_b200 import configs as cf
    from paper_1211_0393_b200.slab import SlabRun
    O = _orc_threads
    c = cf.CONFIGS[cfg]
    f, g, taps = cf.make_problem(c, n=n)
    ref = O.landweber(taps, g, d=O.build_tikhonov(taps, c.alpha, n, n), f_true=f, max_iters=iters,
                      keep_iterates=True)
    dev = torch.device("cuda", 0)
    run = SlabRun(n, P, taps, c.q, c.alpha, rank=-1, device=0)
    try:
        assert run.separable == (cfg == "C5")
        out, h = run.run(torch.from_numpy(g).to(dev), torch.from_numpy(f).to(dev), iters, keep_iterates=True)
        assert h["iterations_executed"] == ref["iterations_executed"]
        assert h["best_iteration"] == ref["best_iteration"]
        np.testing.assert_allclose(h["residual_history"], ref["residual_history"], rtol=1e-10, atol=0)
        np.testing.assert_allclose(h["rre_history"], ref["rre_history"], rtol=1e-10, atol=0)
        for k in range(1, iters + 1):
            x = h["iterates"][k - 1].cpu().numpy()
            e = np.linalg.norm(x - ref["iterates"][k - 1]) / np.linalg.norm(ref["iterates"][k - 1])
            assert e <= 1e-10, (k, e)
        best = ref["iterates"][ref["best_iteration"] - 1]
        assert np.linalg.norm(out.cpu().numpy() - best) / np.linalg.norm(best) <= 1e-10
    finally:
        run.close()


@pytest.mark.gpu
def test_cpp_slab_loop_stopping_rules(dbx, _orc_threads):
    """Fixed iterations without a true image, and the residual rule (the loop
    keeps launching after the stop; every kernel then sees the done flag)."""
    from paper_1211_0393_b200 import configs as cf
    from paper_1211_0393_b200.slab import SlabRun
    O = _orc_threads
    c = cf.CONFIGS["C5"]
    n = 128
    f, g, taps = cf.make_problem(c, n=n)
    dev = torch.device("cuda", 0)
    gt = torch.from_numpy(g).to(dev)
    run = SlabRun(n, 2, taps, c.q, c.alpha, rank=-1, device=0)
    try:
        ref = O.landweber(taps, g, d=O.build_tikhonov(taps, c.alpha, n, n), stop=O.STOP_FIXED, fixed_iters=5)
        out, h = run.run(gt, None, 5)
        assert h["iterations_executed"] == 5 and h["best_iteration"] == 0
        np.testing.assert_allclose(h["residual_history"], ref["residual_history"], rtol=1e-10, atol=0)
        x = out.cpu().numpy()
        assert np.linalg.norm(x - ref["restored"]) / np.linalg.norm(ref["restored"]) <= 1e-10
        eps = ref["residual_history"][2] / np.linalg.norm(g) * 1.0000001
        ref2 = O.landweber(taps, g, d=O.build_tikhonov(taps, c.alpha, n, n), stop=O.STOP_RESID, max_iters=10,
                           resid_eps=eps)
        out2, h2 = run.run(gt, None, 10, resid_eps=eps)
        assert h2["iterations_executed"] == ref2["iterations_executed"] == 3
        x2 = out2.cpu().numpy()
        assert np.linalg.norm(x2 - ref2["restored"]) / np.linalg.norm(ref2["restored"]) <= 1e-10
        with pytest.raises(ValueError, match="zero true image"):
            run.run(gt, torch.zeros_like(gt), 2)
    finally:
        run.close()


@pytest.mark.gpu
def test_nccl_comm_single_rank(dbx):
    """libnccl resolves at run time and a one-rank communicator drives a
    one-slab run (rank 0 of 1: no exchange is issued, the path is the
    NCCL-rank code path)."""
    import ctypes as C

    from paper_1211_0393_b200 import configs as cf
    from paper_1211_0393_b200.slab import SlabRun
    L = dbx.lib()
    uid = (C.c_ubyte * 128)()
    assert L.dbx_comm_unique_id(uid) == 0, L.dbx_last_error()
    h = C.c_void_p()
    assert L.dbx_comm_init(1, uid, 0, 0, C.byref(h)) == 0, L.dbx_last_error()

    class _Comm:
        handle = h
    try:
        c = cf.CONFIGS["C5"]
        f, g, taps = cf.make_problem(c, n=128)
        dev = torch.device("cuda", 0)
        a = SlabRun(128, 1, taps, c.q, c.alpha, rank=0, comm=_Comm(), device=0)
        b = SlabRun(128, 1, taps, c.q, c.alpha, rank=-1, device=0)
        try:
            ga, fa = torch.from_numpy(g).to(dev), torch.from_numpy(f).to(dev)
            xa, ha = a.run(ga, fa, 4)
            xb, hb = b.run(ga, fa, 4)
            assert torch.equal(xa, xb) and ha["rre_history"] == hb["rre_history"]
        finally:
            a.close()
            b.close()
    finally:
        L.dbx_comm_destroy(h)


def test_slab_create_without_device_fails_loudly(dbx):
    """No sm_100 device (this CPU box): the C++ slab loop refuses with a device
    error, there is no CPU fallback."""
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_1211_0393_b200 import configs as cf
    from paper_1211_0393_b200.slab import SlabRun
    c = cf.CONFIGS["C5"]
    _, _, taps = cf.make_problem(c, n=64)
    with pytest.raises(dbx.DeviceError):
        SlabRun(64, 2, taps, c.q, c.alpha, rank=-1, device=0)
