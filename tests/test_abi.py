"""CPU checks of the drop-in boundary: libdbx.so loads, exports every symbol
include/dbx.h declares, validates arguments like the reference, runs the
host-side generators, and REFUSES to compute without a device (no CPU
fallback)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dbx.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dbx_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_path(dbx):
    syms = declared_symbols()
    for must in ("dbx_plan_create", "dbx_blur_apply", "dbx_precond_build", "dbx_precond_apply",
                 "dbx_tensor_apply", "dbx_landweber_run", "dbx_last_error", "dbx_plan_destroy"):
        assert must in syms


def test_library_exports_every_declared_symbol(dbx):
    lib = C.CDLL(dbx.LIB_PATH)
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_no_cpu_fallback_without_device(dbx):
    if dbx.lib().dbx_device_count() > 0:
        pytest.skip("a device is present")
    t = np.full((3, 3), 1.0 / 9)
    with pytest.raises(dbx.DeviceError):
        dbx.BlurOperator(dbx.Psf(t), dbx.BoundaryCondition.AntiReflective, 8, 8)


def test_plan_argument_validation(dbx):
    L = dbx.lib()
    h = C.c_void_p()
    bad = np.full((3, 3), 0.2)  # sums to 1.8
    assert L.dbx_plan_create(8, 8, 1, dbx._ptr(bad), 1, 1, 3, 0, C.byref(h)) == dbx.DBX_EINVAL
    assert "sum to 1" in L.dbx_last_error().decode()
    ok = np.full((3, 3), 1.0 / 9)
    assert L.dbx_plan_create(8, 8, 1, dbx._ptr(ok), 1, 1, 1, 0, C.byref(h)) == dbx.DBX_EINVAL  # Periodic
    tall = np.full((5, 3), 1.0 / 15)
    assert L.dbx_plan_create(1, 8, 1, dbx._ptr(tall), 2, 1, 2, 0, C.byref(h)) == dbx.DBX_EINVAL  # Reflective, q > n
    assert "reflective support condition" in L.dbx_last_error().decode()
    big = np.full((9, 9), 1.0 / 81)
    assert L.dbx_plan_create(5, 5, 1, dbx._ptr(big), 4, 4, 3, 0, C.byref(h)) == dbx.DBX_EINVAL
    assert "support condition" in L.dbx_last_error().decode()
    neg = np.array([[0.5, -0.1, 0.6]])
    assert L.dbx_plan_create(1, 8, 1, dbx._ptr(neg), 0, 1, 3, 0, C.byref(h)) == dbx.DBX_EINVAL
    with pytest.raises(ValueError):
        dbx.Psf(np.ones((2, 3)) / 6)
    with pytest.raises(ValueError):
        dbx.StoppingRule.fixed(-1)
    with pytest.raises(ValueError):
        dbx.StoppingRule.residual_below(0.0)


def test_host_generators_and_noise_match_oracle(dbx, oracle):
    from paper_1211_0393_b200 import configs as cf
    rng = np.random.default_rng(3)
    g = rng.uniform(0, 1, (17, 23))
    for lvl, seed in ((0.01, 99), (0.001, 1), (0.0, 5)):
        assert np.array_equal(dbx.add_noise(g, dbx.NoiseSpec(lvl, seed)), oracle.add_noise(g, lvl, seed))
    for name, c in cf.CONFIGS.items():
        t = cf.make_psf(c)
        assert t.shape == (2 * c.q + 1, 2 * c.q + 1)
        assert abs(t.sum() - 1.0) <= 1e-12 and t.min() >= 0
        oracle.psf_check if hasattr(oracle, "psf_check") else None
    f, gg, taps = cf.make_problem(cf.CONFIGS["C1"], n=64)
    # Honest generation: g is the noiseless direct correlation of the scene plus
    # exactly 1% noise (experiment.hpp:85-93, image.hpp:79-81)
    c = cf.CONFIGS["C1"]
    canvas = 64 + 2 * (2 * c.q + 1)
    scene = np.empty((canvas, canvas))
    dbx._check(dbx.lib().dbx_gen_scene(canvas, canvas, c.shapes, c.sinus_amp, cf.scene_seed(c, 0), dbx._ptr(scene)))
    off = (canvas - 64) // 2
    assert np.array_equal(f, scene[off:off + 64, off:off + 64])
    clean = np.zeros((64, 64))
    q = c.q
    for s1 in range(-q, q + 1):
        for s2 in range(-q, q + 1):
            clean += taps[q + s1, q + s2] * scene[off - s1:off - s1 + 64, off - s2:off - s2 + 64]
    assert abs(np.linalg.norm(gg - clean) / np.linalg.norm(clean) - c.noise) <= 1e-12


def test_mt19937_64_boxmuller_known_answer(oracle):
    """image.hpp:38-66 pins 'mt19937_64-boxmuller-1'.  Independent pure-Python
    mt19937_64 (the C++ standard fixes its 10000th output for the default seed
    5489 at 9981545732273789042) drives a Box-Muller restatement that must match
    the oracle's add_noise draw for draw."""
    class MT64:
        def __init__(self, seed):
            self.mt = [0] * 312
            self.mt[0] = seed & 0xFFFFFFFFFFFFFFFF
            for i in range(1, 312):
                self.mt[i] = (6364136223846793005 * (self.mt[i - 1] ^ (self.mt[i - 1] >> 62)) + i) & 0xFFFFFFFFFFFFFFFF
            self.i = 312

        def __call__(self):
            if self.i >= 312:
                for k in range(312):
                    x = (self.mt[k] & 0xFFFFFFFF80000000) | (self.mt[(k + 1) % 312] & 0x7FFFFFFF)
                    xa = x >> 1
                    if x & 1:
                        xa ^= 0xB5026F5AA96619E9
                    self.mt[k] = self.mt[(k + 156) % 312] ^ xa
                self.i = 0
            y = self.mt[self.i]
            self.i += 1
            y ^= (y >> 29) & 0x5555555555555555
            y ^= (y << 17) & 0x71D67FFFEDA60000
            y ^= (y << 37) & 0xFFF7EEE000000000
            y ^= y >> 43
            return y & 0xFFFFFFFFFFFFFFFF

    m = MT64(5489)
    for _ in range(9999):
        m()
    assert m() == 9981545732273789042
    seed, n = 4242, 10
    m = MT64(seed)
    eta = []
    while len(eta) < n:
        u1 = ((m() >> 11) + 1.0) * 2.0 ** -53
        u2 = (m() >> 11) * 2.0 ** -53
        r = np.sqrt(-2.0 * np.log(u1))
        a = 2.0 * 3.141592653589793 * u2
        eta += [r * np.cos(a), r * np.sin(a)]
    eta = np.array(eta[:n])
    g = np.linspace(1.0, 2.0, n)[None, :]
    want = g + (0.01 * np.linalg.norm(g) / np.linalg.norm(eta)) * eta
    got = oracle.add_noise(g, 0.01, seed)
    assert np.abs(got - want).max() <= 1e-15


def _shim_binary():
    import subprocess
    subprocess.run(["make", "-s", "-C", os.path.join(ROOT, "tests", "cpp")], check=True)
    return os.path.join(ROOT, "tests", "cpp", "build", "shim_test")


def test_cpp_shim_compiles_against_the_c_abi(dbx):
    assert os.path.exists(_shim_binary())


@pytest.mark.gpu
def test_cpp_shim_runs_on_gpu(dbx):
    import subprocess
    r = subprocess.run([_shim_binary()], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "OK", (r.stdout, r.stderr)
