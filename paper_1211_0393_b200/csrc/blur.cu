// blur.cu — K1/K2: anti-reflective blur A x and reblur A' r as a direct FP64
// stencil with the AR extension evaluated on the fly (no padded image).
//
// Replaces (reference, /root/reference/proj/include/deblur/):
//   pad + extend_axis AR branch  boundary.hpp:56-62, 88-102
//   correlate_valid_direct       blur.hpp:39-52
//   apply / apply_reblur_adjoint blur.hpp:75-90
//
// Data layout: one CTA owns a TH x TW output tile of one image; it stages the
// (TH+2q1) x (TW+2q2) AR-extended input window and the oriented mask in shared
// memory, then every thread accumulates R rows x 2 columns (columns lane and
// lane+32 so a warp's shared-memory reads are contiguous, conflict-free).
// Epilogues fuse the solver's vector work: r = g - A x with its ||r||^2
// partial, or x_k = x_{k-1} + tau*A'r with ||x||^2 and ||x-f||^2 partials.
#include <cuda_runtime.h>

#include "../../include/dbx.h"
#include "dbx_internal.h"

namespace dbx {

namespace {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kTW = 64;  // tile width (2 columns per lane)
constexpr int kR = 4;    // rows per thread
constexpr int kTH = kWarps * kR;  // 32

// AR extension of FOV row i (0 <= i < n1) at column j in [-q2, n2+q2):
// f_{-k} = 2 f_0 - f_k, f_{n-1+k} = 2 f_{n-1} - f_{n-1-k}  (boundary.hpp:58-61)
// Reflective (bc = 2, boundary.hpp:49-55): f_{-k} = f_{k-1}, f_{n-1+k} = f_{n-k}.
__device__ __forceinline__ double hext(const double* __restrict__ x, int i, int j, int n2, int bc) {
  const double* row = x + (size_t)i * n2;
  if (bc == DBX_BC_REFLECTIVE) {
    if (j < 0) return row[-j - 1];
    if (j >= n2) return row[2 * n2 - 1 - j];
    return row[j];
  }
  if (j < 0) return 2.0 * row[0] - row[-j];
  if (j >= n2) return 2.0 * row[n2 - 1] - row[2 * (n2 - 1) - j];
  return row[j];
}

// Padded value with the reference's association: rows (axis 2) extended
// first, then columns over the widened image (boundary.hpp:93-100).
__device__ __forceinline__ double pext(const double* __restrict__ x, int i, int j, int n1, int n2, int bc) {
  if (bc == DBX_BC_REFLECTIVE) {
    if (i < 0) return hext(x, -i - 1, j, n2, bc);
    if (i >= n1) return hext(x, 2 * n1 - 1 - i, j, n2, bc);
    return hext(x, i, j, n2, bc);
  }
  if (i < 0) return 2.0 * hext(x, 0, j, n2, bc) - hext(x, -i, j, n2, bc);
  if (i >= n1) return 2.0 * hext(x, n1 - 1, j, n2, bc) - hext(x, 2 * (n1 - 1) - i, j, n2, bc);
  return hext(x, i, j, n2, bc);
}

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kWarps; ++i) s += red[i];
  return s;  // valid in thread 0
}

__global__ void __launch_bounds__(kThreads) blur_ar_kernel(BlurArgs a) {
  DBX_PDL_WAIT();
  const int b = blockIdx.z;
  if (a.st && a.st[b].done) return;
  extern __shared__ double smem[];
  const int q1 = a.q1, q2 = a.q2, n1 = a.n1, n2 = a.n2;
  const int wq = 2 * q2 + 1, hq = 2 * q1 + 1;
  const int pitch = kTW + 2 * q2;
  const int rows = kTH + 2 * q1;
  double* S = smem;
  double* W = smem + (size_t)rows * pitch;
  double* red = W + hq * wq;

  const size_t N = (size_t)n1 * n2;
  const double* x = resolve_ptr(a.x, a.st, a.xsel, b, a.batch, N);
  const int r0 = blockIdx.y * kTH, c0 = blockIdx.x * kTW;

  for (int i = threadIdx.x; i < hq * wq; i += kThreads) W[i] = a.w[i];
  for (int idx = threadIdx.x; idx < rows * pitch; idx += kThreads) {
    const int ti = idx / pitch, tj = idx - ti * pitch;
    const int i = r0 - q1 + ti, j = c0 - q2 + tj;
    double v = 0.0;
    if (i < n1 + q1 && j < n2 + q2) v = pext(x, i, j, n1, n2, a.bc);
    S[idx] = v;
  }
  __syncthreads();

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double acc[kR][2];
#pragma unroll
  for (int i = 0; i < kR; ++i) acc[i][0] = acc[i][1] = 0.0;

  const int band = warp * kR;
  for (int rr = 0; rr < kR + 2 * q1; ++rr) {
    const double* srow = S + (size_t)(band + rr) * pitch + lane;
    for (int u = 0; u < wq; ++u) {
      const double v0 = srow[u], v1 = srow[u + 32];
#pragma unroll
      for (int i = 0; i < kR; ++i) {
        const int t = rr - i;
        if (t >= 0 && t < hq) {
          const double w = W[t * wq + u];
          acc[i][0] = fma(w, v0, acc[i][0]);
          acc[i][1] = fma(w, v1, acc[i][1]);
        }
      }
    }
  }

  double p0 = 0.0, p1 = 0.0;
  const double* g = a.mode == BLUR_RESID ? a.g + (size_t)b * N : nullptr;
  const double* xo = a.mode == BLUR_AXPY ? resolve_ptr(a.xold, a.st, a.xoldsel, b, a.batch, N) : nullptr;
  const double* f = (a.mode == BLUR_AXPY && a.f) ? a.f + (size_t)b * N : nullptr;
  double* y = const_cast<double*>(resolve_ptr(a.y, a.st, a.ysel, b, a.batch, N));
#pragma unroll
  for (int i = 0; i < kR; ++i) {
    const int r = r0 + band + i;
    if (r >= n1) continue;
#pragma unroll
    for (int c2 = 0; c2 < 2; ++c2) {
      const int c = c0 + lane + 32 * c2;
      if (c >= n2) continue;
      const size_t o = (size_t)r * n2 + c;
      const double v = acc[i][c2];
      if (a.mode == BLUR_STORE) {
        y[o] = v;
      } else if (a.mode == BLUR_RESID) {
        const double rv = g[o] - v;
        y[o] = rv;
        p0 += rv * rv;
      } else {
        const double xv = xo[o] + a.tau * v;
        y[o] = xv;
        p0 += xv * xv;
        if (f) {
          const double e = xv - f[o];
          p1 += e * e;
        }
      }
    }
  }
  if (a.mode != BLUR_STORE && a.part.p) {
    const int cta = blockIdx.y * gridDim.x + blockIdx.x;
    double* P = a.part.p + (size_t)b * NUM_SLOTS * a.part.cap;
    const double s0 = block_sum(p0, red);
    if (a.mode == BLUR_RESID) {
      if (threadIdx.x == 0) P[SLOT_R2 * a.part.cap + cta] = s0;
    } else {
      if (threadIdx.x == 0) P[SLOT_X2 * a.part.cap + cta] = s0;
      const double s1 = block_sum(p1, red);
      if (threadIdx.x == 0) P[SLOT_XF2 * a.part.cap + cta] = s1;
    }
  }
}

}  // namespace

void launch_blur(const BlurArgs& a, cudaStream_t s, int* ctas_per_image) {
  dim3 grid((a.n2 + kTW - 1) / kTW, (a.n1 + kTH - 1) / kTH, a.batch);
  const size_t smem =
      sizeof(double) * ((size_t)(kTH + 2 * a.q1) * (kTW + 2 * a.q2) +
                        (size_t)(2 * a.q1 + 1) * (2 * a.q2 + 1) + kWarps);
  static AttrOnce attr;
  attr.ensure(blur_ar_kernel, 227 * 1024);
  if (ctas_per_image) *ctas_per_image = grid.x * grid.y;
  launch_k(blur_ar_kernel, grid, kThreads, smem, s, a);
}

}  // namespace dbx
