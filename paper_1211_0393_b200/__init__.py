"""paper_1211_0393_b200 — B200-native anti-reflective preconditioned Landweber.

Python mirror of the reference ``deblur`` C++ operator API for the AR hot path
(/root/reference/proj/include/deblur): the same names, argument meaning and
error behaviour, implemented over the C-ABI in ``include/dbx.h`` (``libdbx.so``,
sm_100a CUDA kernels).  There is no CPU compute path: every numerical entry
point fails with ``DeviceError`` when no sm_100 device (or the built library)
is present.

Reference correspondences:
  Psf, symmetrize, rotate180          psf.hpp:13-91
  BlurOperator, apply,
  apply_reblur_adjoint                blur.hpp:17-90
  tensor_apply                        transforms.hpp:198-226
  PreconditionerSpec, FilteredOperator,
  build_tikhonov, precondition_apply  preconditioner.hpp:17-90
  StoppingRule, SolverConfig, RestorationRun, SolverDivergence,
  landweber, d_landweber,
  semiconvergence_report              solver.hpp:17-160
  add_noise, rre, NoiseSpec           image.hpp:31-91
"""
from __future__ import annotations

import ctypes as C
import dataclasses
import enum
import os
from typing import List, Optional

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DBX_LIB", os.path.join(_HERE, "libdbx.so"))  # DBX_LIB: A/B builds

DBX_OK, DBX_EINVAL, DBX_EDIVERGED, DBX_ECUDA = 0, 1, 2, 3


class DeviceError(RuntimeError):
    """CUDA / device failure (DBX_ECUDA).  Raised instead of falling back to CPU."""


class SolverDivergence(RuntimeError):
    """solver.hpp:42-44."""


_lib = None


def lib():
    """Loads libdbx.so; raises DeviceError if it was not built."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise DeviceError(f"libdbx.so not built ({LIB_PATH}); run python -m paper_1211_0393_b200.build")
        L = C.CDLL(LIB_PATH)
        vp, i, d = C.c_void_p, C.c_int, C.c_double
        L.dbx_last_error.restype = C.c_char_p
        L.dbx_version.restype = C.c_char_p
        L.dbx_device_count.restype = i
        L.dbx_plan_create.argtypes = [i, i, i, vp, i, i, i, i, C.POINTER(vp)]
        L.dbx_plan_destroy.argtypes = [vp]
        L.dbx_plan_destroy.restype = None
        L.dbx_plan_stream.argtypes = [vp]
        L.dbx_plan_stream.restype = vp
        L.dbx_plan_set_conv.argtypes = [vp, i]
        L.dbx_plan_set_dst.argtypes = [vp, i]
        L.dbx_plan_engines.argtypes = [vp, C.POINTER(i), C.POINTER(i)]
        L.dbx_plan_pipeline.argtypes = [vp, C.POINTER(i)]
        L.dbx_plan_separable.argtypes = [vp, C.POINTER(i), C.POINTER(d)]
        L.dbx_plan_set_fusion.argtypes = [vp, i]
        L.dbx_blur_apply.argtypes = [vp, vp, vp, i]
        L.dbx_precond_build.argtypes = [vp, d]
        L.dbx_precond_eigs.argtypes = [vp, vp]
        L.dbx_precond_set_eigs.argtypes = [vp, vp]
        L.dbx_precond_apply.argtypes = [vp, vp, vp]
        L.dbx_tensor_apply.argtypes = [vp, i, vp, vp]
        L.dbx_landweber_run.argtypes = [vp, vp, vp, d, i, i, i, d, i, vp, vp, vp, vp, vp, vp]
        L.dbx_cgls_run.argtypes = [vp, vp, vp, i, i, i, d, i, vp, vp, vp, vp, vp, vp]
        L.dbx_landweber_run_chunks.argtypes = [vp, i, vp, vp, d, i, i, i, d, i, vp, vp, vp, vp, vp]
        L.dbx_plan_set_timing.argtypes = [vp, i]
        L.dbx_plan_kernel_times.argtypes = [vp, vp, vp, i]
        L.dbx_plan_kernel_profile.argtypes = [vp, i, C.c_char_p, i, C.POINTER(d), C.POINTER(i)]
        L.dbx_plan_launch_count.argtypes = [vp]
        L.dbx_plan_launch_count.restype = C.c_int64
        L.dbx_gen_scene.argtypes = [i, i, i, d, C.c_uint64, vp]
        L.dbx_gen_psf_gaussian.argtypes = [i, i, d, d, d, d, d, vp]
        L.dbx_gen_psf_motion.argtypes = [i, i, d, d, d, vp]
        L.dbx_gen_honest.argtypes = [vp, i, i, vp, i, i, i, i, d, C.c_uint64, i, vp, vp]
        L.dbx_gen_scene_shapes.argtypes = [i, i, i, C.c_uint64, vp]
        L.dbx_mt19937_64_host.argtypes = [C.c_uint64, C.c_uint64, vp]
        L.dbx_mt19937_64_device.argtypes = [C.c_uint64, C.c_uint64, vp, i]
        L.dbx_gen_honest_device.argtypes = [i, i, i, d, C.c_uint64, vp, i, i, i, i, d, C.c_uint64, vp, vp, i]
        L.dbx_add_noise.argtypes = [vp, i, i, d, C.c_uint64, vp]
        L.dbx_precond_build_sweep.argtypes = [vp, vp]
        L.dbx_slab_blur.argtypes = [vp, vp, vp, i, vp, C.POINTER(d)]
        L.dbx_slab_rows.argtypes = [vp, i, vp, vp, i, vp, vp, d, C.POINTER(d)]
        L.dbx_precond_block.argtypes = [vp, i, i, d, i, i, i, i, i, vp]
        L.dbx_transpose.argtypes = [vp, vp, vp, i, i]
        L.dbx_slab_extend.argtypes = [vp, vp, vp, vp, vp]
        L.dbx_slab_pack.argtypes = [vp, vp, vp, i, i]
        # C++ row-slab loop (NCCL communicators, dbx_slab_*)
        L.dbx_comm_unique_id.argtypes = [vp]
        L.dbx_comm_init.argtypes = [i, vp, i, i, C.POINTER(vp)]
        L.dbx_comm_wrap.argtypes = [vp, i, i, C.POINTER(vp)]
        L.dbx_comm_destroy.argtypes = [vp]
        L.dbx_comm_destroy.restype = None
        L.dbx_slab_create.argtypes = [i, i, i, vp, i, i, d, vp, i, C.POINTER(vp)]
        L.dbx_slab_run.argtypes = [vp, vp, vp, d, i, i, d, vp, vp, vp, vp, vp]
        L.dbx_slab_info.argtypes = [vp, C.POINTER(i), C.POINTER(i), C.POINTER(i), C.POINTER(C.c_int64)]
        L.dbx_slab_stream.argtypes = [vp]
        L.dbx_slab_stream.restype = vp
        L.dbx_slab_set_iterates.argtypes = [vp, vp, i]
        L.dbx_slab_destroy.argtypes = [vp]
        L.dbx_slab_destroy.restype = None
        _lib = L
    return _lib


def _check(st: int):
    if st == DBX_OK:
        return
    msg = lib().dbx_last_error().decode()
    if st == DBX_EINVAL:
        raise ValueError(msg)
    if st == DBX_EDIVERGED:
        raise SolverDivergence(msg)
    raise DeviceError(msg)


def _ptr(a):
    """Pointer of a numpy array (host) or a torch CUDA tensor (device)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        if a.is_cuda:
            # libdbx runs on its plans' own non-blocking streams: whatever torch
            # still has queued for this tensor (fills, copies, clones) on its
            # current stream must land before a C-ABI kernel touches the memory
            import torch
            st = torch.cuda.current_stream(a.device)
            if not st.query():
                st.synchronize()
        return C.c_void_p(a.data_ptr())
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    if hasattr(a, "data_ptr"):  # torch tensor: must already be float64 contiguous
        if str(a.dtype) != "torch.float64" or not a.is_contiguous():
            raise ValueError("tensor arguments must be contiguous float64")
        return a
    return np.ascontiguousarray(a, dtype=np.float64)


def _empty_like(a, shape=None):
    if hasattr(a, "data_ptr"):
        import torch
        return torch.empty(shape if shape is not None else a.shape, dtype=torch.float64, device=a.device)
    return np.empty(shape if shape is not None else a.shape)


# ---------------------------------------------------------------------------
# enums (reference order)
# ---------------------------------------------------------------------------
class BoundaryCondition(enum.IntEnum):  # boundary.hpp:9
    Zero = 0
    Periodic = 1
    Reflective = 2
    AntiReflective = 3


class TransformKind(enum.IntEnum):  # transforms.hpp:17
    Dft = 0
    CosineIII = 1
    SineI = 2
    AntiReflective = 3
    AntiReflectiveInverse = 4


class Algebra(enum.IntEnum):  # spectral.hpp:12
    Circulant = 0
    CosineIII = 1
    Tau = 2
    AntiReflective = 3


class ConvEngine(enum.IntEnum):
    Auto = 0
    Direct = 1
    Fft = 2
    FftDense = 3  # FFT engine with the full 2D kernel spectrum even for a rank-1 mask


class DstEngine(enum.IntEnum):
    Auto = 0
    Dense = 1
    Fft = 2
    Rader = 3


# ---------------------------------------------------------------------------
# Psf (psf.hpp:13-46) — host-side mask container and validation
# ---------------------------------------------------------------------------
class Psf:
    kMassTol = 1e-12

    def __init__(self, taps):
        t = np.ascontiguousarray(taps, dtype=np.float64)
        if t.ndim != 2 or t.shape[0] % 2 != 1 or t.shape[1] % 2 != 1:
            raise ValueError("Psf: taps must have odd dimensions")
        if not np.all(np.isfinite(t)):
            raise ValueError("Psf: taps must be finite")
        if np.any(t < 0):
            raise ValueError("Psf: taps must be nonnegative")
        if abs(float(np.sum(t)) - 1.0) > self.kMassTol:
            raise ValueError("Psf: taps must sum to 1 (within 1e-12)")
        self._t = t
        self.q1 = (t.shape[0] - 1) // 2
        self.q2 = (t.shape[1] - 1) // 2

    def taps(self):
        return self._t

    def tap(self, i1, i2):  # psf.hpp:32
        return self._t[self.q1 + i1, self.q2 + i2]


def delta_psf(q1=0, q2=0) -> Psf:  # psf.hpp:41-46
    t = np.zeros((2 * q1 + 1, 2 * q2 + 1))
    t[q1, q2] = 1.0
    return Psf(t)


def symmetrize(p: Psf) -> Psf:  # psf.hpp:71-85
    q1, q2, t = p.q1, p.q2, p.taps()
    s = np.empty_like(t)
    for i1 in range(q1 + 1):
        for i2 in range(q2 + 1):
            avg = (t[q1 - i1, q2 - i2] + t[q1 - i1, q2 + i2] + t[q1 + i1, q2 - i2] + t[q1 + i1, q2 + i2]) / 4.0
            s[q1 + i1, q2 + i2] = s[q1 - i1, q2 + i2] = s[q1 + i1, q2 - i2] = s[q1 - i1, q2 - i2] = avg
    return Psf(s)


def rotate180(p: Psf) -> Psf:  # psf.hpp:88-91
    return Psf(p.taps()[::-1, ::-1])


# ---------------------------------------------------------------------------
# BlurOperator (blur.hpp:17-34) — owns one device plan
# ---------------------------------------------------------------------------
class _Plan:
    def __init__(self, n1, n2, batch, taps, q1, q2, device=0, bc=None):
        self.h = C.c_void_p()
        bc = BoundaryCondition.AntiReflective if bc is None else bc
        _check(lib().dbx_plan_create(n1, n2, batch, _ptr(taps), q1, q2, int(bc), device, C.byref(self.h)))

    def __del__(self):
        try:
            if self.h:
                lib().dbx_plan_destroy(self.h)
        except Exception:
            pass


class BlurOperator:
    """A_n for AntiReflective BCs over a batch of n1 x n2 images."""

    def __init__(self, psf: Psf, bc: BoundaryCondition, n1: int, n2: int, batch: int = 1, device: int = 0):
        if n1 < 1 or n2 < 1:
            raise ValueError("BlurOperator: empty field of view")
        if bc not in (BoundaryCondition.AntiReflective, BoundaryCondition.Reflective):
            raise ValueError("BlurOperator: this path implements AntiReflective and Reflective BCs")
        if bc == BoundaryCondition.Reflective:
            if not (psf.q1 <= n1 and psf.q2 <= n2):
                raise ValueError("reflective support condition violated (q > n)")
        elif not ((psf.q1 == 0 or psf.q1 <= n1 - 2) and (psf.q2 == 0 or psf.q2 <= n2 - 2)):
            raise ValueError("anti-reflective support condition violated (q > n-2)")
        self._psf, self._bc, self.n1, self.n2, self.batch = psf, bc, n1, n2, batch
        self._plan = _Plan(n1, n2, batch, psf.taps(), psf.q1, psf.q2, device, bc)

    def psf(self):
        return self._psf

    def bc(self):
        return self._bc

    @property
    def handle(self):
        return self._plan.h

    def set_conv(self, engine: ConvEngine):
        _check(lib().dbx_plan_set_conv(self.handle, int(engine)))
        return self

    def set_dst(self, engine: DstEngine):
        _check(lib().dbx_plan_set_dst(self.handle, int(engine)))
        return self

    def set_fusion(self, on: bool):
        _check(lib().dbx_plan_set_fusion(self.handle, int(bool(on))))
        return self

    def engines(self):
        c, d = C.c_int(), C.c_int()
        _check(lib().dbx_plan_engines(self.handle, C.byref(c), C.byref(d)))
        return ConvEngine(c.value), DstEngine(d.value)

    def separable(self):
        """(True if the FFT column pass runs the rank-1 separable stencil,
        max |w - a b^T| / max |w| of the mask's best rank-1 factorisation)."""
        f, r = C.c_int(), C.c_double()
        _check(lib().dbx_plan_separable(self.handle, C.byref(f), C.byref(r)))
        return bool(f.value), float(r.value)

    def pipeline_fused(self) -> bool:
        """True when the last landweber run used the fused row pipelines."""
        f = C.c_int()
        _check(lib().dbx_plan_pipeline(self.handle, C.byref(f)))
        return bool(f.value)

    def stream(self):
        return lib().dbx_plan_stream(self.handle)

    def set_timing(self, on: bool):
        _check(lib().dbx_plan_set_timing(self.handle, int(bool(on))))

    def kernel_times(self):
        ms = (C.c_double * 8)()
        cnt = (C.c_int * 8)()
        n = lib().dbx_plan_kernel_times(self.handle, ms, cnt, 8)
        return [float(ms[i]) for i in range(n)], [int(cnt[i]) for i in range(n)]

    def launch_count(self) -> int:
        return int(lib().dbx_plan_launch_count(self.handle))

    def _shape_ok(self, x):
        want = (self.n1, self.n2) if self.batch == 1 else (self.batch, self.n1, self.n2)
        if tuple(x.shape) != want and not (self.batch == 1 and tuple(x.shape) == (1, self.n1, self.n2)):
            raise ValueError("apply: image does not match the operator's field of view")


def apply(op: BlurOperator, f):
    """g = A f (blur.hpp:75-83)."""
    f = _f64(f)
    op._shape_ok(f)
    y = _empty_like(f)
    _check(lib().dbx_blur_apply(op.handle, _ptr(f), _ptr(y), 0))
    return y


def apply_reblur_adjoint(op: BlurOperator, r):
    """A' r with the 180-rotated mask (blur.hpp:87-90)."""
    r = _f64(r)
    op._shape_ok(r)
    y = _empty_like(r)
    _check(lib().dbx_blur_apply(op.handle, _ptr(r), _ptr(y), 1))
    return y


def tensor_apply(kind: TransformKind, x, op: Optional[BlurOperator] = None, engine: DstEngine = DstEngine.Auto):
    """2D separable transform, columns then rows (transforms.hpp:198-226)."""
    x = _f64(x)
    if kind == TransformKind.Dft:
        raise ValueError("tensor_apply: Dft is complex, use dft2_forward")
    n1, n2 = x.shape[-2], x.shape[-1]
    if kind in (TransformKind.AntiReflective, TransformKind.AntiReflectiveInverse) and (n1 < 3 or n2 < 3):
        raise ValueError("tensor_apply: anti-reflective transform needs sizes >= 3")
    if op is None:
        op = _transform_op(n1, n2, 1 if x.ndim == 2 else x.shape[0])
    op.set_dst(engine)
    y = _empty_like(x)
    _check(lib().dbx_tensor_apply(op.handle, int(kind), _ptr(x), _ptr(y)))
    return y


_TOPS = {}


def _transform_op(n1, n2, batch):
    key = (n1, n2, batch)
    if key not in _TOPS:
        _TOPS[key] = BlurOperator(delta_psf(), BoundaryCondition.AntiReflective, n1, n2, batch)
    return _TOPS[key]


# ---------------------------------------------------------------------------
# Preconditioner (preconditioner.hpp:17-90)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class PreconditionerSpec:
    algebra: Algebra = Algebra.AntiReflective
    alpha: float = 0.0


class FilteredOperator:
    """D = T diag(d) T~ (AntiReflective) or R^T diag(d) R (CosineIII); ``eigs``
    is the d grid (sop.eigs), ``source_psf`` the symmetrised mask it came from."""

    def __init__(self, eigs, source_psf, alpha, op, algebra=Algebra.AntiReflective):
        self.eigs = eigs
        self.source_psf = source_psf
        self.alpha = alpha
        self.algebra = algebra
        self.n1, self.n2 = eigs.shape
        self._op = op


_ALGEBRA_BC = {Algebra.AntiReflective: BoundaryCondition.AntiReflective,
               Algebra.CosineIII: BoundaryCondition.Reflective}


def build_tikhonov(p: Psf, spec: PreconditionerSpec, n1: int, n2: int, batch: int = 1) -> FilteredOperator:
    """preconditioner.hpp:62-85: the symmetrised mask's AR or CosineIII (reflective) spectrum, filtered."""
    if spec.algebra not in _ALGEBRA_BC:
        raise ValueError("build_tikhonov: this path implements the AntiReflective and CosineIII algebras")
    if spec.alpha < 0:
        raise ValueError("tikhonov_filter: alpha must be nonnegative")
    src = symmetrize(p)
    op = BlurOperator(p, _ALGEBRA_BC[spec.algebra], n1, n2, batch)
    _check(lib().dbx_precond_build(op.handle, float(spec.alpha)))
    eigs = np.empty((n1, n2))
    _check(lib().dbx_precond_eigs(op.handle, _ptr(eigs)))
    return FilteredOperator(eigs, src, spec.alpha, op, spec.algebra)


def filter_from_eigs(eigs, n1=None, n2=None, batch: int = 1,
                     algebra: Algebra = Algebra.AntiReflective) -> FilteredOperator:
    """A FilteredOperator with an explicit d grid (SpectralOperator{algebra, eigs})."""
    eigs = np.ascontiguousarray(eigs, dtype=np.float64)
    n1, n2 = eigs.shape
    op = BlurOperator(delta_psf(), _ALGEBRA_BC[algebra], n1, n2, batch)
    _check(lib().dbx_precond_set_eigs(op.handle, _ptr(eigs)))
    return FilteredOperator(eigs, None, 0.0, op, algebra)


def precondition_apply(d: FilteredOperator, r, engine: DstEngine = DstEngine.Auto):
    """D r = T (d o T~ r) (preconditioner.hpp:88-90, spectral.hpp:161-165)."""
    r = _f64(r)
    if (r.shape[-2], r.shape[-1]) != (d.n1, d.n2):
        raise ValueError("filter_apply: size mismatch")
    if r.ndim == 3 and r.shape[0] != d._op.batch:
        op = filter_from_eigs(d.eigs, batch=r.shape[0], algebra=d.algebra)._op
    else:
        op = d._op
    op.set_dst(engine)
    y = _empty_like(r)
    _check(lib().dbx_precond_apply(op.handle, _ptr(r), _ptr(y)))
    return y


# ---------------------------------------------------------------------------
# Solver (solver.hpp:17-160)
# ---------------------------------------------------------------------------
class StoppingRuleKind(enum.IntEnum):
    FixedIterations = 0
    MinRre = 1
    RelativeResidualBelow = 2


@dataclasses.dataclass
class StoppingRule:
    kind: StoppingRuleKind = StoppingRuleKind.MinRre
    fixed_iterations: int = 0
    residual_threshold: float = 0.0

    @staticmethod
    def fixed(k: int) -> "StoppingRule":
        if k < 0:
            raise ValueError("StoppingRule: negative iteration count")
        return StoppingRule(StoppingRuleKind.FixedIterations, k, 0.0)

    @staticmethod
    def min_rre() -> "StoppingRule":
        return StoppingRule(StoppingRuleKind.MinRre, 0, 0.0)

    @staticmethod
    def residual_below(eps: float) -> "StoppingRule":
        if not eps > 0.0:
            raise ValueError("StoppingRule: threshold must be positive")
        return StoppingRule(StoppingRuleKind.RelativeResidualBelow, 0, eps)


@dataclasses.dataclass
class SolverConfig:
    tau: float = 1.0
    max_iters: int = 100
    stop: StoppingRule = dataclasses.field(default_factory=StoppingRule.min_rre)
    track_rre_against: Optional[object] = None


@dataclasses.dataclass
class RestorationRun:
    restored: object = None
    iterations_executed: int = 0
    best_iteration: int = 0
    rre_history: List[float] = dataclasses.field(default_factory=list)
    residual_history: List[float] = dataclasses.field(default_factory=list)
    iterates: Optional[np.ndarray] = None


@dataclasses.dataclass
class SemiconvergenceReport:
    best_iter: int = 0
    best_rre: float = 0.0
    diverged_after: bool = False


def _run(op: BlurOperator, d: Optional[FilteredOperator], g, cfg: SolverConfig, keep_iterates=False,
         method: str = "landweber"):
    g = _f64(g)
    op._shape_ok(g)
    f = cfg.track_rre_against
    if f is not None:
        f = _f64(f)
        if tuple(f.shape) != tuple(g.shape):
            raise ValueError("landweber: true image size mismatch")
    if d is not None:
        if (d.n1, d.n2) != (op.n1, op.n2):
            raise ValueError("d_landweber: preconditioner size mismatch")
        if _ALGEBRA_BC.get(d.algebra) != op.bc():
            raise ValueError("d_landweber: preconditioner algebra does not match the BC")
        # the plan keeps one filter grid: always load this operator's (no
        # identity cache: d.eigs may have been edited in place, and object
        # ids are reused after garbage collection)
        _check(lib().dbx_precond_set_eigs(op.handle, _ptr(d.eigs)))
    stop = cfg.stop
    total = stop.fixed_iterations if stop.kind == StoppingRuleKind.FixedIterations else cfg.max_iters
    H = max(total, 1)
    B = op.batch
    on_dev = hasattr(g, "data_ptr")
    restored = _empty_like(g)
    rre_h = np.zeros((B, H))
    res_h = np.zeros((B, H))
    best = (C.c_int * B)()
    done = (C.c_int * B)()
    xh = np.empty((B, H, op.n1, op.n2)) if keep_iterates else None
    if method == "cgls":
        _check(lib().dbx_cgls_run(
            op.handle, _ptr(g), _ptr(f), int(cfg.max_iters), int(stop.kind),
            int(stop.fixed_iterations), float(stop.residual_threshold), 1 if d is not None else 0,
            _ptr(restored), _ptr(rre_h), _ptr(res_h), best, done, _ptr(xh)))
    else:
        _check(lib().dbx_landweber_run(
            op.handle, _ptr(g), _ptr(f), float(cfg.tau), int(cfg.max_iters), int(stop.kind),
            int(stop.fixed_iterations), float(stop.residual_threshold), 1 if d is not None else 0,
            _ptr(restored), _ptr(rre_h), _ptr(res_h), best, done, _ptr(xh)))
    runs = []
    for b in range(B):
        k = done[b]
        runs.append(RestorationRun(
            restored=restored[b] if (g.ndim == 3) else restored,
            iterations_executed=k, best_iteration=best[b],
            rre_history=list(rre_h[b, :k]) if f is not None else [],
            residual_history=list(res_h[b, :k]),
            iterates=xh[b, :k] if xh is not None else None))
    del on_dev
    return runs[0] if g.ndim == 2 else runs


def landweber(op: BlurOperator, g, cfg: SolverConfig, keep_iterates=False):
    """x_{k+1} = x_k + tau A'(g - A x_k) (solver.hpp:139-142)."""
    return _run(op, None, g, cfg, keep_iterates)


def d_landweber(op: BlurOperator, d: FilteredOperator, g, cfg: SolverConfig, keep_iterates=False):
    """x_{k+1} = x_k + tau D A'(g - A x_k) (solver.hpp:145-148)."""
    return _run(op, d, g, cfg, keep_iterates)


def cgls(op: BlurOperator, g, cfg: SolverConfig, d: Optional[FilteredOperator] = None, keep_iterates=False):
    """Reblurred CGLS on min ||A x - g||, preconditioned by D when given
    (config 2's "CGLS-type" iteration; cfg.tau is unused)."""
    return _run(op, d, g, cfg, keep_iterates, method="cgls")


def landweber_chunks(ops, g, cfg: SolverConfig, d: Optional[FilteredOperator] = None):
    """(D-)Landweber of a HOST batch g [B, n1, n2] split over the plans of
    ``ops`` (BlurOperators whose batches sum to B, same size and mask): the
    chunks' uploads and downloads overlap the solves (dbx_landweber_run_chunks;
    page-locked arrays, e.g. torch ``pin_memory()`` tensors, for the overlap).
    Returns one RestorationRun per image, identical to d_landweber/landweber on
    the whole batch."""
    g = _f64(g)
    if hasattr(g, "data_ptr") and g.is_cuda:
        raise ValueError("landweber_chunks: host arrays only")
    B = sum(op.batch for op in ops)
    if g.ndim != 3 or g.shape[0] != B or any((op.n1, op.n2) != tuple(g.shape[1:]) for op in ops):
        raise ValueError("landweber_chunks: g must be [sum of plan batches, n1, n2]")
    f = cfg.track_rre_against
    if f is not None:
        f = _f64(f)
        if tuple(f.shape) != tuple(g.shape):
            raise ValueError("landweber: true image size mismatch")
    if d is not None:
        for op in ops:
            _check(lib().dbx_precond_set_eigs(op.handle, _ptr(d.eigs)))
    stop = cfg.stop
    total = stop.fixed_iterations if stop.kind == StoppingRuleKind.FixedIterations else cfg.max_iters
    H = max(total, 1)
    if hasattr(g, "data_ptr"):
        import torch
        restored = torch.empty(tuple(g.shape), dtype=torch.float64, pin_memory=bool(g.is_pinned()))
    else:
        restored = np.empty(g.shape)
    rre_h = np.zeros((B, H))
    res_h = np.zeros((B, H))
    best = (C.c_int * B)()
    done = (C.c_int * B)()
    handles = (C.c_void_p * len(ops))(*[op.handle for op in ops])
    _check(lib().dbx_landweber_run_chunks(
        handles, len(ops), _ptr(g), _ptr(f), float(cfg.tau), int(cfg.max_iters), int(stop.kind),
        int(stop.fixed_iterations), float(stop.residual_threshold), 1 if d is not None else 0,
        _ptr(restored), _ptr(rre_h), _ptr(res_h), best, done))
    return [RestorationRun(restored=restored[b], iterations_executed=done[b], best_iteration=best[b],
                           rre_history=list(rre_h[b, :done[b]]) if f is not None else [],
                           residual_history=list(res_h[b, :done[b]]), iterates=None) for b in range(B)]


def semiconvergence_report(run: RestorationRun) -> SemiconvergenceReport:  # solver.hpp:152-160
    if len(run.rre_history) == 0:
        raise ValueError("semiconvergence_report: no RRE history")
    h = np.asarray(run.rre_history)
    i = int(np.argmin(h))
    return SemiconvergenceReport(i + 1, float(h[i]), bool(h[-1] > h[i] * 1.05))


# ---------------------------------------------------------------------------
# Image model + synthetic inputs (image.hpp, experiment.hpp:71-99)
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class NoiseSpec:
    relative_level: float = 0.0
    seed: int = 0


kNoiseRngId = "mt19937_64-boxmuller-1"


def add_noise(g, spec: NoiseSpec):
    g = np.ascontiguousarray(g, dtype=np.float64)
    if spec.relative_level < 0:
        raise ValueError("add_noise: negative level")
    out = np.empty_like(g)
    _check(lib().dbx_add_noise(_ptr(g), g.shape[0], g.shape[1], float(spec.relative_level), int(spec.seed), _ptr(out)))
    return out


def rre(x, f_true) -> float:  # image.hpp:85-91 (host helper)
    x, f = np.asarray(x, dtype=np.float64), np.asarray(f_true, dtype=np.float64)
    if x.shape != f.shape:
        raise ValueError("rre: dimension mismatch")
    den = float(np.linalg.norm(f))
    if not den > 0:
        raise ValueError("rre: zero true image")
    return float(np.linalg.norm(x - f)) / den


from . import configs  # noqa: E402  (synthetic BASELINE configs)

__all__ = [n for n in dir() if not n.startswith("_")]
