"""GPU-side Honest synthesis (experiment.hpp:71-99, image.hpp:44-82).

CPU: the shape-parameter export reproduces dbx_gen_scene's draws, and the
host mt19937_64 stream matches the C++-standard known answer.  GPU: the device
mt19937_64 stream equals std::mt19937_64 word for word (lengths around the
312-word block), and dbx_gen_honest_device matches the host generator — f_true
bit for bit, g to rounding (<= 1e-12 relative) — on C1 at full size, on the sinusoid-background C4
scene and on the full 8192^2 C5 canvas (the size the device path exists for)."""
import ctypes as C
import time

import numpy as np
import pytest

from paper_1211_0393_b200 import configs as cf


def _host_stream(dbx, seed, count):
    out = np.empty(count, dtype=np.uint64)
    dbx._check(dbx.lib().dbx_mt19937_64_host(seed, count, dbx._ptr(out)))
    return out


def test_host_stream_known_answer(dbx):
    # C++ [rand.predef]: the 10000th output of a default-constructed mt19937_64
    assert int(_host_stream(dbx, 5489, 10000)[-1]) == 9981545732273789042


def test_shape_params_reproduce_host_scene(dbx):
    """Painting the exported shapes (numpy, same operations) gives the host scene."""
    rows, cols, ns, seed = 70, 90, 25, 77
    L = dbx.lib()
    P = np.empty((ns, 12))
    dbx._check(L.dbx_gen_scene_shapes(rows, cols, ns, seed, dbx._ptr(P)))
    host = np.empty((rows, cols))
    dbx._check(L.dbx_gen_scene(rows, cols, ns, 0.0, seed, dbx._ptr(host)))
    img = np.zeros((rows, cols))
    for p in P:
        r0, r1, c0, c1 = (int(v) for v in p[8:12])
        for r in range(r0, r1 + 1):
            dy = (r + 0.5) - p[1]
            for c in range(c0, c1 + 1):
                dx = (c + 0.5) - p[2]
                u, v = dx * p[5] + dy * p[6], -dx * p[6] + dy * p[5]
                inside = (u * u) / (p[3] * p[3]) + (v * v) / (p[4] * p[4]) <= 1.0 if p[0] else \
                    abs(u) <= p[3] and abs(v) <= p[4]
                if inside:
                    img[r, c] = p[7]
    assert np.array_equal(img, host)


@pytest.mark.gpu
@pytest.mark.parametrize("seed,count", [(5489, 10000), (123456789, 311), (7, 312), (42, 313), (2024, 1 << 20)])
def test_device_mt19937_64_stream(dbx, seed, count):
    dev = np.empty(count, dtype=np.uint64)
    dbx._check(dbx.lib().dbx_mt19937_64_device(seed, count, dbx._ptr(dev), 0))
    assert np.array_equal(dev, _host_stream(dbx, seed, count))


def _compare(cfg, n):
    f_h, g_h, taps_h = cf.make_problem(cfg, n=n)
    t0 = time.perf_counter()
    f_d, g_d, taps_d = cf.make_problem_device(cfg, n=n)
    secs = time.perf_counter() - t0
    assert np.array_equal(taps_h, taps_d)
    if cfg.sinus_amp == 0.0:
        assert np.array_equal(f_h, f_d), "scene / crop must match the host painter bit for bit"
    else:
        # shapes bit for bit; the smooth background through device sin (<= 1 ulp)
        assert np.abs(f_d - f_h).max() <= 4e-16 * (1.0 + np.abs(f_h).max())
    # noise: device libm (<= 1 ulp) and the norm reductions' order (rescale
    # factor level ||g|| / ||eta|| over up to 67M terms) — rounding level
    rel = np.linalg.norm(g_d - g_h) / np.linalg.norm(g_h)
    assert rel <= 1e-12, rel
    return secs


@pytest.mark.gpu
@pytest.mark.parametrize("name,n", [("C1", 256), ("C2", 192), ("C4", 256)])
def test_device_honest_matches_host(dbx, name, n):
    _compare(cf.CONFIGS[name], n)


@pytest.mark.gpu
def test_device_honest_full_c5_canvas(dbx):
    """C5 (8192^2 FOV on an 8254^2 canvas, 2000 shapes): equal to the host
    generator, and generated in well under the host's seconds."""
    c = cf.CONFIGS["C5"]
    cf.make_problem_device(c, n=256)  # warm-up (context, module load)
    secs = _compare(c, c.n)
    assert secs < 5.0, secs


@pytest.mark.gpu
def test_device_honest_into_device_buffers(dbx):
    import torch
    c = cf.CONFIGS["C3"]
    n = 128
    f = torch.empty((n, n), dtype=torch.float64, device="cuda")
    g = torch.empty_like(f)
    cf.make_problem_device(c, n=n, out=(f, g))
    f_h, g_h, _ = cf.make_problem(c, n=n)
    assert np.array_equal(f.cpu().numpy(), f_h)
    assert np.linalg.norm(g.cpu().numpy() - g_h) <= 1e-14 * np.linalg.norm(g_h)


@pytest.mark.gpu
def test_device_honest_refuses_bad_margin(dbx):
    L = dbx.lib()
    taps = np.full((5, 5), 1 / 25)
    f, g = np.empty((60, 60)), np.empty((60, 60))
    st = L.dbx_gen_honest_device(62, 62, 3, 0.0, 1, dbx._ptr(taps), 2, 2, 60, 60, 0.01, 2, dbx._ptr(f),
                                 dbx._ptr(g), 0)
    assert st == 1 and b"margin" in L.dbx_last_error()
