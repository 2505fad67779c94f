// cg.cu — vector kernels of the (preconditioned) reblurred CGLS recurrence
// (config 2's "CGLS-type" iteration).  The reference has
// no CG (SPEC.md:517 lists Krylov methods as a non-goal); the recurrence is
// the standard CGLS / CGNR on min ||A x - g|| with the AR preconditioner D as
// the SPD weight of the normal equations:
//
//   r0 = g, s0 = A' r0, z0 = D s0, p0 = z0, gamma0 = <s0, z0>
//   q = A p;  alpha = gamma / ||q||^2;  x += alpha p;  r -= alpha q
//   s = A' r;  z = D s;  gamma' = <s, z>;  beta = gamma' / gamma;  p = z + beta p
//
// The blurs and D are the path's own kernels; these kernels carry the scalar
// recurrence per image (fixed-order reductions, no float atomics) and fold
// the x / r updates with the norms the finalize kernel books.
#include <cuda_runtime.h>

#include "dbx_internal.h"

namespace dbx {

namespace {

constexpr int kT = 256;

__device__ double block_sum_fixed(double v) {
  __shared__ double red[kT / 32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kT / 32; ++i) s += red[i];
  return s;
}

__device__ double partial_total(const double* p, int cnt) {
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += kT) s += p[i];
  return block_sum_fixed(s);
}

// alpha = gamma / ||q||^2 from the q-blur's ||r||^2 slot (q' = -A p there)
__global__ void cg_alpha_kernel(const ImgState* st, CgScalars* cs, Partials pt, int cnt) {
  DBX_PDL_WAIT();
  const int b = blockIdx.x;
  if (st[b].done) return;
  const double qq = partial_total(pt.p + ((size_t)b * NUM_SLOTS + SLOT_R2) * pt.cap, cnt);
  if (threadIdx.x == 0) cs[b].alpha = qq > 0.0 ? cs[b].gamma / qq : 0.0;
}

// x_nxt = x_cur + alpha p; r += alpha q' (q' = -A p); partials ||x||^2,
// ||x - f||^2, ||r||^2 (finalize slots)
__global__ void cg_update_kernel(const double* X3, const ImgState* st, const CgScalars* cs, const double* p,
                                 const double* qn, double* r, const double* f, int batch, size_t N, Partials pt,
                                 double* x_out) {
  DBX_PDL_WAIT();
  const int b = blockIdx.y;
  if (st[b].done) return;
  const double al = cs[b].alpha;
  const double* xc = X3 + ((size_t)st[b].cur * batch + b) * N;
  double* xn = x_out + ((size_t)st[b].nxt * batch + b) * N;
  const size_t o = (size_t)b * N;
  double sx = 0.0, sf = 0.0, sr = 0.0;
  for (size_t i = (size_t)blockIdx.x * kT + threadIdx.x; i < N; i += (size_t)gridDim.x * kT) {
    const double xv = fma(al, p[o + i], xc[i]);
    xn[i] = xv;
    sx += xv * xv;
    if (f) {
      const double e = xv - f[o + i];
      sf += e * e;
    }
    const double rv = fma(al, qn[o + i], r[o + i]);
    r[o + i] = rv;
    sr += rv * rv;
  }
  double* P = pt.p + (size_t)b * NUM_SLOTS * pt.cap;
  const double a0 = block_sum_fixed(sx);
  if (threadIdx.x == 0) P[SLOT_X2 * pt.cap + blockIdx.x] = a0;
  const double a1 = block_sum_fixed(sf);
  if (threadIdx.x == 0) P[SLOT_XF2 * pt.cap + blockIdx.x] = a1;
  const double a2 = block_sum_fixed(sr);
  if (threadIdx.x == 0) P[SLOT_R2 * pt.cap + blockIdx.x] = a2;
}

// per-block partials of <s, z>
__global__ void cg_dot_kernel(const ImgState* st, const double* s, const double* z, size_t N, double* part,
                              int cap) {
  DBX_PDL_WAIT();
  const int b = blockIdx.y;
  if (st && st[b].done) return;
  const size_t o = (size_t)b * N;
  double acc = 0.0;
  for (size_t i = (size_t)blockIdx.x * kT + threadIdx.x; i < N; i += (size_t)gridDim.x * kT)
    acc = fma(s[o + i], z[o + i], acc);
  const double t = block_sum_fixed(acc);
  if (threadIdx.x == 0) part[(size_t)b * cap + blockIdx.x] = t;
}

// gamma' = sum; beta = gamma' / gamma; gamma = gamma' (init: beta = 0)
__global__ void cg_beta_kernel(const ImgState* st, CgScalars* cs, const double* part, int cap, int cnt, int init) {
  DBX_PDL_WAIT();
  const int b = blockIdx.x;
  if (st[b].done) return;
  const double gn = partial_total(part + (size_t)b * cap, cnt);
  if (threadIdx.x == 0) {
    cs[b].beta = init ? 0.0 : (cs[b].gamma != 0.0 ? gn / cs[b].gamma : 0.0);
    cs[b].gamma = gn;
  }
}

// p = z + beta p
__global__ void cg_xpay_kernel(const ImgState* st, const CgScalars* cs, const double* z, double* p, size_t N) {
  DBX_PDL_WAIT();
  const int b = blockIdx.y;
  if (st[b].done) return;
  const double be = cs[b].beta;
  const size_t o = (size_t)b * N;
  for (size_t i = (size_t)blockIdx.x * kT + threadIdx.x; i < N; i += (size_t)gridDim.x * kT)
    p[o + i] = fma(be, p[o + i], z[o + i]);
}

int grid_x(size_t N, int cap) {
  size_t g = (N + kT - 1) / kT;
  if (g > 1024) g = 1024;
  if ((int)g > cap) g = (size_t)cap;
  return (int)(g < 1 ? 1 : g);
}

}  // namespace

void launch_cg_alpha(const ImgState* st, CgScalars* cs, Partials pt, int cnt, int batch, cudaStream_t s) {
  launch_k(cg_alpha_kernel, batch, kT, 0, s, st, cs, pt, cnt);
}

int launch_cg_update(const double* X3, const ImgState* st, const CgScalars* cs, const double* p, const double* qn,
                     double* r, const double* f, int batch, size_t N, Partials pt, cudaStream_t s) {
  const int gx = grid_x(N, pt.cap);
  launch_k(cg_update_kernel, dim3(gx, batch), kT, 0, s, X3, st, cs, p, qn, r, f, batch, N, pt, const_cast<double*>(X3));
  return gx;
}

int launch_cg_dot(const ImgState* st, const double* a, const double* b, int batch, size_t N, double* part, int cap,
                  cudaStream_t s) {
  const int gx = grid_x(N, cap);
  launch_k(cg_dot_kernel, dim3(gx, batch), kT, 0, s, st, a, b, N, part, cap);
  return gx;
}

void launch_cg_beta(const ImgState* st, CgScalars* cs, const double* part, int cap, int cnt, int init, int batch,
                    cudaStream_t s) {
  launch_k(cg_beta_kernel, batch, kT, 0, s, st, cs, part, cap, cnt, init);
}

void launch_cg_xpay(const ImgState* st, const CgScalars* cs, const double* z, double* p, int batch, size_t N,
                    cudaStream_t s) {
  launch_k(cg_xpay_kernel, dim3(grid_x(N, 1 << 30), batch), kT, 0, s, st, cs, z, p, N);
}

}  // namespace dbx
