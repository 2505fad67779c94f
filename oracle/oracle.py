"""CPU ORACLE wrapper (TEST INFRASTRUCTURE ONLY).

ctypes bindings over ``oracle/build/liborc.so`` (built from
``oracle/deblur_oracle.cpp`` by ``oracle/Makefile``), the scalar C++
restatement of the reference ``deblur`` library's anti-reflective
preconditioned-Landweber path.  Only ``tests/``, ``__graft_entry__.smoke()``
and ``bench.py``'s cpu_baseline / ``--impl reference`` legs may import this
module — it is the checker, never the product.

Function names mirror the reference API (file:line in the C++ source).
Errors map like the reference: invalid arguments raise ``ValueError``
(std::invalid_argument), divergence raises ``OracleDivergence``
(SolverDivergence, solver.hpp:42-44).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "build", "liborc.so")
_lib = None

STOP_FIXED, STOP_MINRRE, STOP_RESID = 0, 1, 2
KIND_SINEI, KIND_AR, KIND_ARINV = 2, 3, 4


class OracleDivergence(RuntimeError):
    pass


def build() -> str:
    subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def gen_lib_path() -> str:
    """Host-only build of the input generators (csrc/gen.cpp), see Makefile."""
    path = os.path.join(_HERE, "build", "liborcgen.so")
    if not os.path.exists(path):
        build()
    return path


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        _lib = C.CDLL(_LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_rre.restype = C.c_double
        _lib.orc_rre.argtypes = [C.c_void_p, C.c_void_p, C.c_long]
        _lib.orc_add_noise.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_double, C.c_uint64, C.c_void_p]
    return _lib


def set_threads(n: int) -> None:
    """Worker threads for the line-parallel 2D passes; results are
    bit-identical for any count (each line's arithmetic is unchanged)."""
    lib().orc_set_threads(int(n))


def get_threads() -> int:
    return int(lib().orc_get_threads())


def set_kernel_cache(on: bool) -> None:
    """Keep the (bit-identical) mask spectrum between correlation calls
    instead of recomputing it as the reference does (blur.hpp:65-66); tests
    use it to shorten long trajectories, timing legs leave it off."""
    lib().orc_set_kernel_cache(int(bool(on)))


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _check(st: int):
    if st == 0:
        return
    msg = lib().orc_last_error().decode()
    if st == 1:
        raise ValueError(msg)
    raise OracleDivergence(msg)


def _q(taps):
    taps = _f64(taps)
    if taps.ndim != 2 or taps.shape[0] % 2 == 0 or taps.shape[1] % 2 == 0:
        raise ValueError("Psf: taps must have odd dimensions")
    return taps, (taps.shape[0] - 1) // 2, (taps.shape[1] - 1) // 2


def fft(x, sign=-1):
    z = np.ascontiguousarray(x, dtype=np.complex128).copy()
    _check(lib().orc_fft(_p(z), C.c_int(z.size), C.c_int(sign)))
    return z


def symmetrize(taps):
    taps, q1, q2 = _q(taps)
    out = np.empty_like(taps)
    _check(lib().orc_symmetrize(_p(taps), q1, q2, _p(out)))
    return out


def rotate180(taps):
    return np.ascontiguousarray(_f64(taps)[::-1, ::-1])


def pad_ar(f, q1, q2):
    f = _f64(f)
    out = np.empty((f.shape[0] + 2 * q1, f.shape[1] + 2 * q2))
    _check(lib().orc_pad_ar(_p(f), f.shape[0], f.shape[1], q1, q2, _p(out)))
    return out


BC_REFLECTIVE, BC_ANTIREFLECTIVE = 2, 3  # BoundaryCondition order, boundary.hpp:9
KIND_COSINE3 = 1  # TransformKind::CosineIII (forward R); -1 in tensor_apply = R^T


def apply(taps, f, adjoint=False, path=0, bc=BC_ANTIREFLECTIVE, long_double=False):
    """blur.hpp:75-83 (adjoint=True: apply_reblur_adjoint, blur.hpp:87-90).
    long_double=True computes in long double (the FP64 rounding floor)."""
    taps, q1, q2 = _q(taps)
    f = _f64(f)
    out = np.empty_like(f)
    if long_double:
        _check(lib().orc_apply_p(_p(taps), q1, q2, _p(f), f.shape[0], f.shape[1], int(adjoint), int(path), bc, 1,
                                 _p(out)))
    elif bc == BC_ANTIREFLECTIVE:
        _check(lib().orc_apply(_p(taps), q1, q2, _p(f), f.shape[0], f.shape[1], int(adjoint), int(path), _p(out)))
    else:
        _check(lib().orc_apply_bc(_p(taps), q1, q2, _p(f), f.shape[0], f.shape[1], int(adjoint), int(path), bc,
                                  _p(out)))
    return out


def cosine3_forward(v, inverse=False):
    """transforms.hpp:88-110 (R_m v, or R_m^T v when inverse)."""
    v = _f64(v)
    y = np.empty_like(v)
    _check(lib().orc_cosine3(int(inverse), _p(v), v.size, _p(y)))
    return y


def sine1_forward(v):
    v = _f64(v)
    y = np.empty_like(v)
    _check(lib().orc_sine1(_p(v), v.size, _p(y)))
    return y


def ar_forward(v):
    v = _f64(v)
    y = np.empty_like(v)
    _check(lib().orc_ar_1d(0, _p(v), v.size, _p(y)))
    return y


def ar_inverse(v):
    v = _f64(v)
    y = np.empty_like(v)
    _check(lib().orc_ar_1d(1, _p(v), v.size, _p(y)))
    return y


def make_ar_transform(m):
    alpha = C.c_double()
    p = np.empty(max(m - 2, 0))
    _check(lib().orc_ar_alpha(m, C.byref(alpha), _p(p)))
    return alpha.value, p


def tensor_apply(kind, x, long_double=False):
    x = _f64(x)
    y = np.empty_like(x)
    _check(lib().orc_tensor_apply_p(kind, _p(x), x.shape[0], x.shape[1], int(bool(long_double)), _p(y)))
    return y


def precondition_apply_ld(taps, alpha, r):
    """D r in long double with the filter rebuilt in long double from the taps."""
    taps, q1, q2 = _q(taps)
    r = _f64(r)
    y = np.empty_like(r)
    _check(lib().orc_precondition_apply_ld(_p(taps), q1, q2, C.c_double(alpha), _p(r), r.shape[0], r.shape[1],
                                           _p(y)))
    return y


def eig_antireflective(taps, n1, n2):
    taps, q1, q2 = _q(taps)
    e = np.empty((n1, n2))
    _check(lib().orc_eig_antireflective(_p(taps), q1, q2, n1, n2, _p(e)))
    return e


def tikhonov_filter(eigs, alpha):
    eigs = _f64(eigs)
    d = np.empty_like(eigs)
    _check(lib().orc_tikhonov_filter(_p(eigs), eigs.shape[0], eigs.shape[1], C.c_double(alpha), _p(d)))
    return d


def build_tikhonov(taps, alpha, n1, n2, bc=BC_ANTIREFLECTIVE):
    """preconditioner.hpp:62-85 (AntiReflective, or CosineIII for reflective BCs)."""
    taps, q1, q2 = _q(taps)
    d = np.empty((n1, n2))
    if bc == BC_ANTIREFLECTIVE:
        _check(lib().orc_build_tikhonov(_p(taps), q1, q2, n1, n2, C.c_double(alpha), _p(d)))
    else:
        _check(lib().orc_build_tikhonov_bc(_p(taps), q1, q2, n1, n2, C.c_double(alpha), bc, _p(d)))
    return d


def precondition_apply(d, r, bc=BC_ANTIREFLECTIVE):
    d, r = _f64(d), _f64(r)
    y = np.empty_like(r)
    if bc == BC_ANTIREFLECTIVE:
        _check(lib().orc_precondition_apply(_p(d), _p(r), r.shape[0], r.shape[1], _p(y)))
    else:
        _check(lib().orc_precondition_apply_bc(_p(d), _p(r), r.shape[0], r.shape[1], bc, _p(y)))
    return y


def add_noise(g, level, seed):
    g = _f64(g)
    out = np.empty_like(g)
    _check(lib().orc_add_noise(_p(g), g.shape[0], g.shape[1], level, seed, _p(out)))
    return out


def rre(x, f):
    x, f = _f64(x), _f64(f)
    return lib().orc_rre(_p(x), _p(f), x.size)


def cgls(taps, g, d=None, f_true=None, max_iters=100, stop=STOP_MINRRE, fixed_iters=0, resid_eps=0.0,
         keep_iterates=False, bc=BC_ANTIREFLECTIVE):
    """Reblurred (preconditioned) CGLS, SURVEY §8f f2 — NOT in the reference
    (SPEC.md:517 lists Krylov methods as a non-goal): the standard CGLS / CGNR
    recurrence on min ||A x - g|| with D as the SPD weight, built from the
    reference's own primitives (apply / apply_reblur_adjoint blur.hpp:75-90,
    precondition_apply preconditioner.hpp:88-90) and its loop bookkeeping
    (solver.hpp:107-124: guard before recording, strict-'<' best, residual
    rule after recording).  Parity of the recurrence itself is unpinned."""
    g = _f64(g)
    total = fixed_iters if stop == STOP_FIXED else max_iters
    ft = _f64(f_true) if f_true is not None else None
    gn = float(np.linalg.norm(g))
    fn = float(np.linalg.norm(ft)) if ft is not None else 0.0
    x = np.zeros_like(g)
    r = g.copy()
    prec = (lambda v: precondition_apply(d, v, bc)) if d is not None else (lambda v: v)
    s = apply(taps, r, adjoint=True, bc=bc)
    z = prec(s)
    gamma = float(np.sum(s * z))
    p = z.copy()
    rre_h, res_h, xs = [], [], []
    best, best_e, k_done = 0, np.inf, 0
    for k in range(1, total + 1):
        q = apply(taps, p, bc=bc)
        qq = float(np.sum(q * q))
        alpha = gamma / qq if qq > 0 else 0.0
        x = x + alpha * p
        r = r - alpha * q
        if gn > 0 and np.linalg.norm(x) > 1e8 * gn:
            raise RuntimeError("landweber: iterate exceeded 1e8 * ||g||")
        rn = float(np.linalg.norm(r))
        res_h.append(rn)
        if ft is not None:
            e = float(np.linalg.norm(x - ft)) / fn
            rre_h.append(e)
            if e < best_e:
                best_e, best = e, k
                x_best = x.copy()
        if keep_iterates:
            xs.append(x.copy())
        k_done = k
        if stop == STOP_RESID and gn > 0 and rn / gn < resid_eps:
            break
        s = apply(taps, r, adjoint=True, bc=bc)
        z = prec(s)
        gnew = float(np.sum(s * z))
        beta = gnew / gamma if gamma != 0 else 0.0
        gamma = gnew
        p = z + beta * p
    restored = x_best if (ft is not None and stop == STOP_MINRRE and best > 0) else x
    return {"restored": restored, "iterations_executed": k_done, "best_iteration": best,
            "rre_history": np.array(rre_h), "residual_history": np.array(res_h),
            "iterates": np.array(xs) if keep_iterates else None}


def landweber(taps, g, d=None, f_true=None, tau=1.0, max_iters=100, stop=STOP_MINRRE,
              fixed_iters=0, resid_eps=0.0, conv_path=0, keep_iterates=False, bc=BC_ANTIREFLECTIVE,
              long_double_alpha=None):
    """solver.hpp:63-148.  Returns a dict shaped like RestorationRun.

    long_double_alpha: run the same loop in long double instead (the FP64
    rounding-floor reference); None -> FP64 oracle,
    a value >= 0 -> D-Landweber with the filter rebuilt in long double for
    that alpha, a negative value -> plain Landweber.  ``d`` must be None then."""
    taps, q1, q2 = _q(taps)
    g = _f64(g)
    n1, n2 = g.shape
    total = fixed_iters if stop == STOP_FIXED else max_iters
    hist = max(total, 1)
    restored = np.empty_like(g)
    rre_h = np.zeros(hist)
    res_h = np.zeros(hist)
    best = C.c_int()
    done = C.c_int()
    xh = np.empty((hist, n1, n2)) if keep_iterates else None
    dd = _f64(d) if d is not None else None
    ft = _f64(f_true) if f_true is not None else None
    if long_double_alpha is not None:
        if dd is not None:
            raise ValueError("landweber: pass either d or long_double_alpha")
        st = lib().orc_landweber_ld(
            _p(taps), q1, q2, n1, n2, C.c_double(long_double_alpha), _p(g), _p(ft) if ft is not None else None,
            C.c_double(tau), max_iters, stop, fixed_iters, C.c_double(resid_eps), conv_path, bc, _p(restored),
            _p(rre_h), _p(res_h), C.byref(best), C.byref(done), _p(xh) if xh is not None else None)
    else:
        st = lib().orc_landweber_bc(
            _p(taps), q1, q2, n1, n2, _p(dd) if dd is not None else None, _p(g),
            _p(ft) if ft is not None else None, C.c_double(tau), max_iters, stop, fixed_iters,
            C.c_double(resid_eps), conv_path, bc, _p(restored), _p(rre_h), _p(res_h), C.byref(best),
            C.byref(done), _p(xh) if xh is not None else None)
    _check(st)
    k = done.value
    return {
        "restored": restored,
        "iterations_executed": k,
        "best_iteration": best.value,
        "rre_history": rre_h[:k].copy() if ft is not None else np.zeros(0),
        "residual_history": res_h[:k].copy(),
        "iterates": xh[:k] if xh is not None else None,
    }


def semiconvergence_report(rre_history):
    """solver.hpp:152-160: (best_iter 1-based at the FIRST minimum — std::min_element
    —, best_rre, diverged_after = last > 1.05 * best).  Raises ValueError on an
    empty history (detail::require)."""
    h = [float(v) for v in rre_history]
    if not h:
        raise ValueError("semiconvergence_report: no RRE history")
    b = 0
    for i in range(1, len(h)):
        if h[i] < h[b]:
            b = i
    return b + 1, h[b], h[-1] > h[b] * 1.05
