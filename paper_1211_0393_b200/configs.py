"""The five BASELINE.json workloads as seeded synthetic problems.

Every config uses Honest data generation (experiment.hpp:71-99): a scene on a
canvas of n + 2(2q+1) pixels per axis (configs[0] names 286 = 256 + 2*15) is
blurred by direct correlation, cropped to the centred FOV, and corrupted by
add_noise (image.hpp:72-82).  Scenes and masks come from the host generators in
csrc/gen.cpp; their exact definitions and the decisions the reference leaves
open (alpha, shape count for C3, motion-tail decay, axis order) are recorded in
DESIGN.md §Synthetic inputs.  These seeded synthetic images stand in for the
paper's Cameraman/Bridge benchmark images, which are not available.
"""
from __future__ import annotations

import dataclasses
from typing import Optional, Tuple

import numpy as np


@dataclasses.dataclass(frozen=True)
class Config:
    name: str
    n: int
    batch: int
    q: int
    psf_kind: str                       # "gauss" | "motion"
    sigma: Tuple[float, float] = (1.0, 1.0)
    theta_deg: float = 0.0
    offset: Tuple[float, float] = (0.0, 0.0)
    motion: Tuple[float, float, float] = (0.0, 0.0, 0.0)  # length, angle, tail
    shapes: int = 20
    sinus_amp: float = 0.0
    noise: float = 0.01
    iters: int = 50
    alpha: float = 0.02
    plain_too: bool = False
    seed: int = 1

    @property
    def canvas(self) -> int:
        return self.n + 2 * (2 * self.q + 1)


CONFIGS = {
    "C1": Config("C1", 256, 1, 7, "gauss", (2.0, 3.0), 0.0, (1.0, -1.0), shapes=20, noise=0.01,
                 iters=50, alpha=0.02, seed=101),
    "C2": Config("C2", 512, 1, 10, "motion", motion=(15.0, 30.0, 3.0), shapes=40, noise=0.005,
                 iters=100, alpha=1.0, plain_too=True, seed=202),
    "C3": Config("C3", 1024, 64, 15, "gauss", (4.0, 4.5), 0.0, (1.0, 0.0), shapes=100, noise=0.01,
                 iters=40, alpha=0.02, seed=303),
    "C4": Config("C4", 2048, 1, 31, "gauss", (8.0, 10.0), 20.0, (2.0, -3.0), shapes=200,
                 sinus_amp=0.2, noise=0.001, iters=30, alpha=0.02, seed=404),
    "C5": Config("C5", 8192, 1, 15, "gauss", (5.0, 3.0), 0.0, (2.0, 1.0), shapes=2000, noise=0.01,
                 iters=20, alpha=0.02, seed=505),
}


_GEN_LIB = None


def use_generator_library(path: Optional[str]) -> None:
    """Generate inputs through another build of csrc/gen.cpp (same source,
    same bytes out).  bench.py's reference arm points this at the oracle's own
    copy (oracle/build/liborcgen.so) so that the CPU-only arm never maps the
    product library libdbx.so; None restores the default."""
    global _GEN_LIB
    if path is None:
        _GEN_LIB = None
        return
    import ctypes as C
    L = C.CDLL(path)
    vp, i, d = C.c_void_p, C.c_int, C.c_double
    L.dbx_gen_scene.argtypes = [i, i, i, d, C.c_uint64, vp]
    L.dbx_gen_psf_gaussian.argtypes = [i, i, d, d, d, d, d, vp]
    L.dbx_gen_psf_motion.argtypes = [i, i, d, d, d, vp]
    L.dbx_gen_honest.argtypes = [vp, i, i, vp, i, i, i, i, d, C.c_uint64, i, vp, vp]
    _GEN_LIB = L


def _gen():
    from . import _ptr, lib
    if _GEN_LIB is not None:
        def check(st):
            if st != 0:
                raise ValueError(f"input generator: invalid argument (status {st})")
        return _GEN_LIB, check, _ptr
    from . import _check
    return lib(), _check, _ptr


def make_psf(cfg: Config, q: Optional[int] = None) -> np.ndarray:
    L, _check, _ptr = _gen()
    q = cfg.q if q is None else q
    t = np.empty((2 * q + 1, 2 * q + 1))
    if cfg.psf_kind == "gauss":
        _check(L.dbx_gen_psf_gaussian(q, q, cfg.sigma[0], cfg.sigma[1], cfg.theta_deg,
                                      cfg.offset[0], cfg.offset[1], _ptr(t)))
    else:
        length, ang, tail = cfg.motion
        _check(L.dbx_gen_psf_motion(q, q, length, ang, tail, _ptr(t)))
    return t


def scene_seed(cfg: Config, image: int) -> int:
    return cfg.seed * 1_000_003 + image


def make_problem(cfg: Config, image: int = 0, n: Optional[int] = None, threads: int = 0):
    """Returns (f_true, g, taps) for one image of the config.  ``n`` overrides
    the FOV size (scaled-down parity cases keep the mask, shapes and noise)."""
    L, _check, _ptr = _gen()
    n = cfg.n if n is None else n
    taps = make_psf(cfg)
    canvas = n + 2 * (2 * cfg.q + 1)
    scene = np.empty((canvas, canvas))
    s = scene_seed(cfg, image)
    _check(L.dbx_gen_scene(canvas, canvas, cfg.shapes, cfg.sinus_amp, s, _ptr(scene)))
    f = np.empty((n, n))
    g = np.empty((n, n))
    _check(L.dbx_gen_honest(_ptr(scene), canvas, canvas, _ptr(taps), cfg.q, cfg.q, n, n,
                            cfg.noise, s ^ 0x5DEECE66D, threads, _ptr(f), _ptr(g)))
    return f, g, taps


def make_problem_device(cfg: Config, image: int = 0, n: Optional[int] = None, device: int = 0, out=None):
    """make_problem's data generated on the GPU (dbx_gen_honest_device, SURVEY
    §8f f4): same seeds, same scene (f_true bit for bit), g to rounding.
    ``out``: optional (f, g) pair of float64 buffers (numpy arrays or
    torch CUDA tensors) to fill in place; else numpy arrays are returned."""
    from . import _check, _ptr, lib
    n = cfg.n if n is None else n
    taps = make_psf(cfg)
    canvas = n + 2 * (2 * cfg.q + 1)
    s = scene_seed(cfg, image)
    if out is None:
        out = (np.empty((n, n)), np.empty((n, n)))
    f, g = out
    _check(lib().dbx_gen_honest_device(canvas, canvas, cfg.shapes, cfg.sinus_amp, s, _ptr(taps), cfg.q, cfg.q,
                                       n, n, cfg.noise, s ^ 0x5DEECE66D, _ptr(f), _ptr(g), int(device)))
    return f, g, taps


def make_batch(cfg: Config, images: int, first: int = 0, n: Optional[int] = None, threads: int = 0):
    n = cfg.n if n is None else n
    F = np.empty((images, n, n))
    G = np.empty((images, n, n))
    taps = None
    for i in range(images):
        f, g, taps = make_problem(cfg, first + i, n, threads)
        F[i], G[i] = f, g
    return F, G, taps
