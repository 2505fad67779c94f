"""Algorithmic work model of the AR path (bytes / flops per kernel launch and
per pixel-iteration), used by bench.py for the roofline fields and by
DESIGN.md §4.

Two accountings are reported:

* per kernel class, the ALGORITHMIC work of the form actually executed
  (nominal 5 N log2 N flops per complex N-point FFT, 8 flops per complex
  multiply-add, 2(2q+1)^2 flops per direct-stencil pixel; bytes = the arrays a
  launch must read and write once);
* the SURVEY §8d canonical step model: B = 72 B / px-it (D-Landweber fused
  dataflow) and F = 4(2q+1)^2 (two dense stencils, as the reference's
  correlate_valid_direct computes them) + 250 (nominal FFT-form DST-I), with
  T_min = max(B W / BW_HBM, F W / P_FP64).
"""
from __future__ import annotations

import math

CONV_LENGTHS = [64, 72, 80, 96, 128, 144, 160, 192, 256, 270, 288, 320, 384, 512, 540, 576, 640, 768,
                1024, 1080, 1152, 1280, 1536, 2048, 2160, 2304, 2560, 3072, 4096, 4320, 4608, 5120,
                6144, 8192, 8640]
DIRECT_DFT = [15, 31, 63, 255, 1023, 4095]
BLUE_LENGTHS = [16, 32, 64, 128, 256, 512, 1024, 2048, 4096, 8192]


def conv_len(n: int, q: int) -> int:
    need = n + 2 * q
    need += need % 2
    for L in CONV_LENGTHS:
        if L >= need:
            return L
    return 0


def dst_line_flops(n: int, packed: bool = True) -> float:
    """Nominal flops of one AR transform line (length n).  The DST-I of the
    interior (N = n-1) is one complex N-point DFT per line, or — packed real
    form (pk_fill / pk_split, two lines per DFT) — half of one; the DFT is
    direct (N smooth) or Bluestein (2 FFTs of M + 3 pointwise passes).
    Pre/post-processing: ~16 flops per element (sine pre-twiddle, split,
    odd-output scan, AR ramp)."""
    N = n - 1
    share = 0.5 if packed else 1.0
    if N in DIRECT_DFT:
        return share * 5.0 * N * math.log2(N) + 16.0 * N
    M = next((m for m in BLUE_LENGTHS if m >= 2 * N - 1), 0)
    if not M:
        return 2.0 * (n - 2) * (n - 2)  # dense form
    return share * (2 * 5.0 * M * math.log2(M) + 3 * 6.0 * M) + 16.0 * N


def row_fft_pass_flops(n1: int, n2: int, q2: int) -> float:
    """One direction of the row FFTs of an FFT-form blur (two real rows per
    complex FFT of length L2)."""
    L2 = conv_len(n2, q2)
    return (n1 + 1) // 2 * 5.0 * L2 * math.log2(L2)


def col_pass_flops(n1: int, n2: int, q1: int, q2: int) -> float:
    """Column pass: Lh columns x (forward FFT L1, spectrum multiply, inverse)."""
    L1, L2 = conv_len(n1, q1), conv_len(n2, q2)
    return (L2 // 2 + 1) * (2 * 5.0 * L1 * math.log2(L1) + 6.0 * L1)


def fused_classes(n: int, q: int, images: int) -> dict:
    """Per-iteration algorithmic work of the fused preconditioned pipeline
    (fused.cu) by timing class, for `images` n x n images.

    bytes = the arrays each launch must read and write once (Z/Y half spectra
    16 n Lh bytes, images 8 n^2 bytes; the shared d^T grid once per launch)."""
    L2 = conv_len(n, q)
    Lh = L2 // 2 + 1
    Z, P = 16.0 * n * Lh, 8.0 * n * n
    rows, cols = row_fft_pass_flops(n, n, q), col_pass_flops(n, n, q, q)
    dst = n * dst_line_flops(n, packed=True)
    return {
        # rows_ainv_tt (inverse rows of A'r + T~ rows), dst_tcols (T~ cols, d, T cols),
        # rows_t_axpy_afwd (T rows + axpy + forward rows of A x)
        "ar_transform_pass": {"launches": 3, "flops": images * (4 * dst + 2 * rows),
                              "bytes": images * (2 * Z + 7 * P) + P},
        # conv_col(A) + rows_ainv_resid (inverse rows of A x, r = g - A x, forward rows of r)
        "blur(A)+residual": {"launches": 2, "flops": images * (cols + 2 * rows), "bytes": images * (4 * Z + P)},
        # conv_col(A')
        "blur_adjoint(A')": {"launches": 1, "flops": images * cols, "bytes": images * 2 * Z},
    }


def fused_sep_classes(n: int, q: int, images: int) -> dict:
    """Same for the separable pipeline of a rank-1 mask (fused.cu *_sep,
    spectral.cu cols_sep_real): the blurs are direct row / column
    correlations, 2(2q+1) flops per pixel per axis; every intermediate is a
    real n x n array (8 n^2 bytes)."""
    P = 8.0 * n * n
    stencil = 2.0 * (2 * q + 1) * n * n
    dst = n * dst_line_flops(n, packed=True)
    return {
        # rows_tt_sep (A'r rows -> T~ rows), dst_tcols (T~ cols, d, T cols),
        # rows_t_axpy_sep (T rows + axpy + row pass of A x)
        "ar_transform_pass": {"launches": 3, "flops": images * (4 * dst + stencil), "bytes": images * 9 * P + P},
        # cols_sep_real(A) + rows_resid_sep (r = g - A x, row pass of A' r)
        "blur(A)+residual": {"launches": 2, "flops": images * (2 * stencil + 2.0 * n * n), "bytes": images * 5 * P},
        # cols_sep_real(A')
        "blur_adjoint(A')": {"launches": 1, "flops": images * stencil, "bytes": images * 2 * P},
    }


def fused_sep_kernels(n: int, q: int, images: int) -> dict:
    """Per-kernel, per-launch algorithmic work of the separable fused
    pipeline (the C3 bench path), keyed by the launcher names dbx_api.cu
    reports through dbx_plan_kernel_profile ("name#class").  Bytes per
    pixel per image (8-byte reals, every array read / written once):

      cols_sep_real (A')  Z'^T -> Y' = A'r                      16
      rows_tt_sep         Y' -> T~ rows -> u^T                   16
      dst_tcols           u^T -> T~ cols, x d, T cols -> s       16 (+ d once per launch)
      rows_t_axpy_sep     s, x_{k-1}, f -> x_k, Z^T (row pass)   40
      cols_sep_real (A)   Z^T -> Y = A x_k                       16
      rows_resid_sep      Y, g -> r (norm), Z'^T (row pass)      24
    """
    P = 8.0 * n * n
    stencil = 2.0 * (2 * q + 1) * n * n
    dst = n * dst_line_flops(n, packed=True)
    return {
        "cols_sep_real#0": {"bytes": images * 2 * P, "flops": images * stencil},
        "rows_tt_sep#2": {"bytes": images * 2 * P, "flops": images * dst},
        "dst_tcols#2": {"bytes": images * 2 * P + P, "flops": images * 2 * dst},
        "rows_t_axpy_sep#2": {"bytes": images * 5 * P, "flops": images * (dst + stencil + 4.0 * n * n)},
        "cols_sep_real#1": {"bytes": images * 2 * P, "flops": images * stencil},
        "rows_resid_sep#1": {"bytes": images * 3 * P, "flops": images * (stencil + 2.0 * n * n)},
    }


def conv_apply_flops(n1: int, n2: int, q1: int, q2: int) -> float:
    L1, L2 = conv_len(n1, q1), conv_len(n2, q2)
    Lh = L2 // 2 + 1
    rows = (n1 + 1) // 2 * 2 * 5.0 * L2 * math.log2(L2)          # fwd + inv row FFTs (packed pairs)
    cols = Lh * (2 * 5.0 * L1 * math.log2(L1) + 6.0 * L1)       # fwd, multiply, inv
    return rows + cols


def conv_apply_bytes(n1: int, n2: int, q1: int, q2: int, epi_arrays: int) -> float:
    L2 = conv_len(n2, q2)
    Lh = L2 // 2 + 1
    z = 16.0 * n1 * Lh
    return 8.0 * n1 * n2 + z + 2 * z + z + 8.0 * n1 * n2 * epi_arrays


def direct_apply_flops(n1: int, n2: int, q1: int, q2: int) -> float:
    return 2.0 * (2 * q1 + 1) * (2 * q2 + 1) * n1 * n2


def transform_iteration_flops(n1: int, n2: int, packed: bool = True) -> float:
    """Four AR transform passes (T~ rows/cols, T cols/rows) per iteration."""
    return 2 * n1 * dst_line_flops(n2, packed) + 2 * n2 * dst_line_flops(n1, packed)


def transform_iteration_bytes(n1: int, n2: int) -> float:
    # rows T~: r+w 16; cols (T~, d, T): r+w + d = 24; rows T + axpy: r v, x, f, w x = 32
    return (16 + 24 + 32) * float(n1 * n2)


def canonical(q: int, px_it: float, seconds: float, bw_gbs: float, p_fp64_tflops: float):
    """Speed-of-light of the reference's own algorithm: dense
    direct-stencil correlation for A and A' plus FFT-form DST-I.  The FFT-form
    pipeline does far fewer flops, so t_meas < t_min is possible."""
    B, F = 72.0, 4.0 * (2 * q + 1) ** 2 + 250.0
    t_min = max(B * px_it / (bw_gbs * 1e9), F * px_it / (p_fp64_tflops * 1e12))
    return {"bytes_per_px_it": B, "flops_per_px_it": F, "t_min_s": t_min, "t_meas_s": seconds,
            "t_min_over_t_meas": t_min / seconds if seconds > 0 else None,
            "bound": "fp64" if F * bw_gbs * 1e9 > B * p_fp64_tflops * 1e12 else "hbm"}
