// solver_kernels.cu — K5 (Tikhonov filter grid) and K6 (deterministic norm
// reductions, history recording, best-iterate tracking, stopping rules).
//
// Replaces (reference):
//   symbol_real                  psf.hpp:98-109
//   antireflective_grid / eig_antireflective   spectral.hpp:63-69, 120-133
//   tikhonov_filter              preconditioner.hpp:37-57
//   landweber_loop bookkeeping   solver.hpp:86-130 (guard, histories, strict-'<'
//                                best, residual rule), rre image.hpp:85-91
#include <cuda_runtime.h>
#include <math.h>

#include "dbx_internal.h"
#include "finalize.cuh"

namespace dbx {

namespace {

constexpr double kPi = 3.141592653589793238462643383279502884;

// cos(s * x_r) tables on the AR grid x_0 = 0, x_r = r*pi/(n-1), x_{n-1} = 0
// (spectral.hpp:63-69); argument formed exactly like the reference
// (double(r)*kPi/double(n-1), then s*x) so both sides see the same angle.
// grid 1: the reflective (DCT-III) grid x_r = r pi / n (spectral.hpp:50-54)
__global__ void cos_table_kernel(int n, int q, double* tab, int grid) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n * (q + 1)) return;
  const int r = idx / (q + 1), s = idx - r * (q + 1);
  double x = 0.0;
  if (grid == 1) x = (double)r * kPi / (double)n;
  else if (r >= 1 && r <= n - 2) x = (double)r * kPi / (double)(n - 1);
  tab[idx] = cos((double)s * x);
}

// d(a,b) = 1 / (lambda^2 + alpha), lambda = symbol_real(h_sym, x_a, x_b) with
// the reference accumulation order: h00, axis-1 terms, axis-2 terms, cross.
// Block [r0, r0+nr) x [c0, c0+nc) of the n1 x n2 grid; out row-major
// (nr x nc), or transposed (nc x nr) when tr (a rank's d^T block for the
// column pass of a row-slab decomposition).
__global__ void filter_kernel(const double* __restrict__ h, int q1, int q2, int n1, int n2,
                              const double* __restrict__ c1, const double* __restrict__ c2,
                              double alpha, double* __restrict__ d, int* zero_flag,
                              int r0, int nr, int c0, int nc, int tr) {
  extern __shared__ double hs[];
  const int wq = 2 * q2 + 1;
  for (int i = threadIdx.x; i < (2 * q1 + 1) * wq; i += blockDim.x) hs[i] = h[i];
  __syncthreads();
  const int bl = blockIdx.x * blockDim.x + threadIdx.x;
  const int bcol = c0 + bl;
  const int arow = r0 + blockIdx.y;
  if (bl >= nc) return;
  const double* C1 = c1 + (size_t)arow * (q1 + 1);
  const double* C2 = c2 + (size_t)bcol * (q2 + 1);
  auto tap = [&](int s1, int s2) { return hs[(q1 + s1) * wq + (q2 + s2)]; };
  double acc = tap(0, 0);
  for (int s1 = 1; s1 <= q1; ++s1) acc += 2.0 * tap(s1, 0) * C1[s1];
  for (int s2 = 1; s2 <= q2; ++s2) acc += 2.0 * tap(0, s2) * C2[s2];
  for (int s1 = 1; s1 <= q1; ++s1) {
    const double a1 = C1[s1];
    for (int s2 = 1; s2 <= q2; ++s2) acc += 4.0 * tap(s1, s2) * a1 * C2[s2];
  }
  const double m2 = acc * acc;
  if (!(m2 > 0.0)) atomicOr(zero_flag, 1);
  const size_t at = tr ? (size_t)bl * nr + blockIdx.y : (size_t)blockIdx.y * nc + bl;
  d[at] = 1.0 / (m2 + alpha);
}

// Fixed-order block reduction (deterministic).
__device__ double block_reduce(double v) {
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
  return s;
}

__device__ double strided_sumsq(const double* p, size_t n) {
  double s = 0.0;
  for (size_t i = threadIdx.x; i < n; i += blockDim.x) s += p[i] * p[i];
  return block_reduce(s);
}

// ||g||, ||f|| (solver.hpp:73-74, image.hpp:85-91) as a two-level fixed-order
// reduction: grid (K, batch) CTAs each reduce one contiguous chunk into the
// partials buffer, then one CTA per image sums its K partials in index order
// (deterministic; a single CTA per image left 148-SM HBM idle: 59 ms for one
// 8192^2 image).
__global__ void norms_partial_kernel(const double* g, const double* f, size_t N, size_t chunk, Partials pt) {
  DBX_PDL_WAIT();
  const int b = blockIdx.y, k = blockIdx.x;
  const size_t lo = (size_t)k * chunk, n = lo < N ? (N - lo < chunk ? N - lo : chunk) : 0;
  const double gs = strided_sumsq(g + (size_t)b * N + lo, n);
  const double fs = f ? strided_sumsq(f + (size_t)b * N + lo, n) : 0.0;
  if (threadIdx.x == 0) {
    double* P = pt.p + (size_t)b * NUM_SLOTS * pt.cap;
    P[SLOT_X2 * pt.cap + k] = gs;
    P[SLOT_XF2 * pt.cap + k] = fs;
  }
}

__global__ void norms_init_kernel(Partials pt, int cnt, int has_f, ImgState* st) {
  DBX_PDL_WAIT();
  const int b = blockIdx.x;
  const double* P = pt.p + (size_t)b * NUM_SLOTS * pt.cap;
  double gs = 0.0, fs = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) gs += P[SLOT_X2 * pt.cap + i];
  gs = block_reduce(gs);
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) fs += P[SLOT_XF2 * pt.cap + i];
  fs = block_reduce(fs);
  if (threadIdx.x == 0) {
    st[b].g_norm = sqrt(gs);
    st[b].f_norm = has_f ? sqrt(fs) : 0.0;
  }
}

__global__ void state_init_kernel(ImgState* st, int batch) {
  DBX_PDL_WAIT();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= batch) return;
  ImgState s = st[b];
  s.cur = 0;
  s.best = 0;
  s.nxt = 1;
  s.done = 0;
  s.iters = 0;
  s.best_iter = 0;
  s.diverged_at = 0;
  s.best_rre = INFINITY;
  st[b] = s;
}

__device__ double partial_sum(const double* p, int cnt) {
  double s = 0.0;
  for (int i = threadIdx.x; i < cnt; i += blockDim.x) s += p[i];
  return block_reduce(s);
}

// One CTA per image: finalize.cuh finalize_image.
__global__ void finalize_kernel(FinalizeArgs a) {
  DBX_PDL_WAIT();
  finalize_image(a, blockIdx.x);
}

__global__ void select_copy_kernel(const double* X3, const ImgState* st, int which_best,
                                   int batch, size_t N, double* out) {
  DBX_PDL_WAIT();
  const int b = blockIdx.y;
  const int idx = (which_best && st[b].best_iter > 0) ? st[b].best : st[b].cur;
  const double* src = X3 + ((size_t)idx * batch + b) * N;
  double* dst = out + (size_t)b * N;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N;
       i += (size_t)gridDim.x * blockDim.x)
    dst[i] = src[i];
}

// out[c][r] = in[r][c] through a 32 x 33 shared tile (coalesced both ways).
__global__ void transpose_kernel(const double* __restrict__ in, double* __restrict__ out, int rows, int cols) {
  DBX_PDL_WAIT();
  __shared__ double tile[32][33];
  const int c0 = blockIdx.x * 32, r0 = blockIdx.y * 32;
  const size_t img = (size_t)blockIdx.z * rows * cols;  // batch of matrices
  in += img;
  out += img;
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i, c = c0 + threadIdx.x;
    if (r < rows && c < cols) tile[i][threadIdx.x] = in[(size_t)r * cols + c];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int c = c0 + i, r = r0 + threadIdx.x;
    if (r < rows && c < cols) out[(size_t)c * rows + r] = tile[threadIdx.x][i];
  }
}

// Global AR extension rows of a slab (boundary.hpp:58-61 along axis 1):
// top: ext[i] = 2 x[0] - x[q - i] (i < q); bottom: ext[q + rows + k - 1] =
// 2 x[rows-1] - x[rows-1-k] (k = 1..q).
__global__ void slab_ar_rows_kernel(const double* __restrict__ x, double* __restrict__ ext, int rows, int n2,
                                    int q, int top, int bot) {
  DBX_PDL_WAIT();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y + 1;  // 1..q
  if (c >= n2) return;
  if (top) ext[(size_t)(q - k) * n2 + c] = 2.0 * x[c] - x[(size_t)k * n2 + c];
  if (bot) ext[(size_t)(q + rows + k - 1) * n2 + c] = 2.0 * x[(size_t)(rows - 1) * n2 + c] - x[(size_t)(rows - 1 - k) * n2 + c];
}


// ---- C++ row-slab loop (dbx_slab_run) -----------------------------------
// Global AR rows of the first / last slab into separate halo buffers (the
// separable slab blur reads halos in place): top[q - k] = 2 x[0] - x[k],
// bot[k - 1] = 2 x[rows-1] - x[rows-1-k], k = 1..q (boundary.hpp:56-64).
__global__ void slab_ar_halo_kernel(const double* __restrict__ x, int rows, int n2, int q, double* top, double* bot) {
  DBX_PDL_WAIT();
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  const int k = blockIdx.y + 1;
  if (c >= n2) return;
  if (top) top[(size_t)(q - k) * n2 + c] = 2.0 * x[c] - x[(size_t)k * n2 + c];
  if (bot) bot[(size_t)(k - 1) * n2 + c] = 2.0 * x[(size_t)(rows - 1) * n2 + c] - x[(size_t)(rows - 1 - k) * n2 + c];
}

// sum of squares of the slab's g and f: per-CTA partials (slots X2 / XF2)
__global__ void slab_sumsq_kernel(const double* g, const double* f, size_t n, size_t chunk, Partials pt) {
  DBX_PDL_WAIT();
  const size_t lo = (size_t)blockIdx.x * chunk, m = lo < n ? (n - lo < chunk ? n - lo : chunk) : 0;
  const double gs = strided_sumsq(g + lo, m);
  const double fs = f ? strided_sumsq(f + lo, m) : 0.0;
  if (threadIdx.x == 0) {
    pt.p[SLOT_X2 * pt.cap + blockIdx.x] = gs;
    pt.p[SLOT_XF2 * pt.cap + blockIdx.x] = fs;
  }
}

// fixed-order sums of the slab's partial slots into tot[0..2]
__global__ void slab_tot_kernel(Partials pt, int cnt_x, int cnt_r, int track, double* tot, const ImgState* st) {
  DBX_PDL_WAIT();
  if (st && st->done) return;
  const double x2 = partial_sum(pt.p + SLOT_X2 * pt.cap, cnt_x);
  const double xf2 = track ? partial_sum(pt.p + SLOT_XF2 * pt.cap, cnt_x) : 0.0;
  const double r2 = cnt_r > 0 ? partial_sum(pt.p + SLOT_R2 * pt.cap, cnt_r) : 0.0;
  if (threadIdx.x == 0) {
    tot[0] = x2;
    tot[1] = xf2;
    tot[2] = r2;
  }
}

// in-process ranks (LocalWorld analogue): tot_p <- sum over p in rank order
__global__ void slab_local_allreduce_kernel(double* tots, int parts, int stride) {
  DBX_PDL_WAIT();
  const int i = threadIdx.x;
  if (i >= 3) return;
  double s = 0.0;
  for (int p = 0; p < parts; ++p) s += tots[(size_t)p * stride + i];
  for (int p = 0; p < parts; ++p) tots[(size_t)p * stride + i] = s;
}

__global__ void slab_state_init_kernel(ImgState* st, const double* tot2) {
  DBX_PDL_WAIT();
  ImgState s;
  s.cur = s.best = s.nxt = 0;
  s.done = 0;
  s.iters = 0;
  s.best_iter = 0;
  s.diverged_at = 0;
  s.pad_ = 0;
  s.best_rre = INFINITY;
  s.g_norm = sqrt(tot2[0]);
  s.f_norm = sqrt(tot2[1]);
  *st = s;
}

// The loop bookkeeping of finalize_kernel on the all-reduced norms (every
// rank holds the same totals, so every rank takes the same decisions).
// s.best = 1 marks "x_k is the new best" for slab_best_copy_kernel.
__global__ void slab_finalize_kernel(ImgState* st, const double* tot, int k, double* rre_hist, double* res_hist,
                                     int track, int stop_kind, double eps) {
  DBX_PDL_WAIT();
  ImgState s = *st;
  s.best = 0;
  if (s.done) { *st = s; return; }
  const double xn = sqrt(tot[0]);
  if (xn > 1e8 * s.g_norm && s.g_norm > 0.0) {  // solver.hpp:107-108
    s.done = 2;
    s.diverged_at = k;
    *st = s;
    return;
  }
  const double rn = sqrt(tot[2]);
  if (res_hist) res_hist[k - 1] = rn;
  if (track) {
    const double e = sqrt(tot[1]) / s.f_norm;
    if (rre_hist) rre_hist[k - 1] = e;
    if (e < s.best_rre) {  // strict '<' (solver.hpp:114)
      s.best_rre = e;
      s.best_iter = k;
      s.best = 1;
    }
  }
  s.iters = k;
  if (stop_kind == 2 && s.g_norm > 0.0 && rn / s.g_norm < eps) s.done = 1;
  *st = s;
}

__global__ void slab_best_copy_kernel(const ImgState* st, const double* __restrict__ x, double* __restrict__ best,
                                      size_t n) {
  DBX_PDL_WAIT();
  if (!st->best) return;
  const double2* x2 = reinterpret_cast<const double2*>(x);
  double2* b2 = reinterpret_cast<double2*>(best);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n / 2; i += (size_t)gridDim.x * blockDim.x)
    b2[i] = x2[i];
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) best[n - 1] = x[n - 1];
}

__global__ void zero_kernel(double* p, size_t n) {
  DBX_PDL_WAIT();
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (size_t)gridDim.x * blockDim.x)
    p[i] = 0.0;
}

}  // namespace

void launch_build_filter(const double* sym_taps, int q1, int q2, int n1, int n2, double alpha,
                         double* d, int* zero_flag, cudaStream_t s, int grid) {
  launch_build_filter_block(sym_taps, q1, q2, n1, n2, alpha, 0, n1, 0, n2, 0, d, zero_flag, s, grid);
}

void launch_build_filter_block(const double* sym_taps, int q1, int q2, int n1, int n2, double alpha, int r0,
                               int nr, int c0, int nc, int tr, double* d, int* zero_flag, cudaStream_t s,
                               int grid) {
  double *c1 = nullptr, *c2 = nullptr;
  cudaMallocAsync(&c1, sizeof(double) * (size_t)n1 * (q1 + 1), s);
  cudaMallocAsync(&c2, sizeof(double) * (size_t)n2 * (q2 + 1), s);
  cos_table_kernel<<<(n1 * (q1 + 1) + 255) / 256, 256, 0, s>>>(n1, q1, c1, grid);
  cos_table_kernel<<<(n2 * (q2 + 1) + 255) / 256, 256, 0, s>>>(n2, q2, c2, grid);
  const size_t sm = sizeof(double) * (2 * q1 + 1) * (2 * q2 + 1);
  if (sm > 48 * 1024)
    cudaFuncSetAttribute(filter_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
  dim3 fgrid((nc + 127) / 128, nr);
  filter_kernel<<<fgrid, 128, sm, s>>>(sym_taps, q1, q2, n1, n2, c1, c2, alpha, d, zero_flag, r0, nr, c0, nc, tr);
  cudaFreeAsync(c1, s);
  cudaFreeAsync(c2, s);
}

void launch_norms_init(const double* g, const double* f, int batch, size_t N, ImgState* st, Partials pt,
                       cudaStream_t s) {
  // ~4 resident 512-thread CTAs per SM over the whole batch, chunks >= 16 K elements
  size_t K = (size_t)(4 * 148 + batch - 1) / batch;
  const size_t kmax = (N + 16383) / 16384;
  if (K > kmax) K = kmax;
  if (K > (size_t)pt.cap) K = pt.cap;
  if (K < 1) K = 1;
  const size_t chunk = (N + K - 1) / K;
  launch_k(norms_partial_kernel, dim3((unsigned)K, batch), 512, 0, s, g, f, N, chunk, pt);
  launch_k(norms_init_kernel, batch, 256, 0, s, pt, (int)K, f != nullptr, st);
}

void launch_finalize(const FinalizeArgs& a, cudaStream_t s) {
  launch_k(finalize_kernel, a.batch, 256, 0, s, a);
}

void launch_state_init(ImgState* st, int batch, cudaStream_t s) {
  launch_k(state_init_kernel, (batch + 127) / 128, 128, 0, s, st, batch);
}

void launch_select_copy(const double* X3, const ImgState* st, int which_best, int batch,
                        size_t N, double* out, cudaStream_t s) {
  dim3 grid((unsigned)((N + 255) / 256 < 1024 ? (N + 255) / 256 : 1024), batch);
  launch_k(select_copy_kernel, grid, 256, 0, s, X3, st, which_best, batch, N, out);
}

void launch_transpose(const double* in, double* out, int rows, int cols, cudaStream_t s, int batch) {
  dim3 grid((cols + 31) / 32, (rows + 31) / 32, batch);
  launch_k(transpose_kernel, grid, dim3(32, 8), 0, s, in, out, rows, cols);
}

void launch_slab_ar_rows(const double* x, double* ext, int rows, int n2, int q, int top, int bot, cudaStream_t s) {
  if (q <= 0 || !(top || bot)) return;
  dim3 grid((n2 + 255) / 256, q);
  launch_k(slab_ar_rows_kernel, grid, 256, 0, s, x, ext, rows, n2, q, top, bot);
}


void launch_slab_ar_halo(const double* x, int rows, int n2, int q, double* top, double* bot, cudaStream_t s) {
  if (q <= 0 || !(top || bot)) return;
  dim3 grid((n2 + 255) / 256, q);
  launch_k(slab_ar_halo_kernel, grid, 256, 0, s, x, rows, n2, q, top, bot);
}
int launch_slab_sumsq(const double* g, const double* f, size_t n, Partials pt, cudaStream_t s) {
  int k = (int)((n + (1 << 20) - 1) >> 20);
  k = k < 1 ? 1 : (k > pt.cap ? pt.cap : k);
  const size_t chunk = (n + k - 1) / k;
  launch_k(slab_sumsq_kernel, k, 256, 0, s, g, f, n, chunk, pt);
  return k;
}
void launch_slab_tot(Partials pt, int cnt_x, int cnt_r, int track, double* tot, const ImgState* st, cudaStream_t s) {
  launch_k(slab_tot_kernel, 1, 256, 0, s, pt, cnt_x, cnt_r, track, tot, st);
}
void launch_slab_local_allreduce(double* tots, int parts, int stride, cudaStream_t s) {
  launch_k(slab_local_allreduce_kernel, 1, 32, 0, s, tots, parts, stride);
}
void launch_slab_state_init(ImgState* st, const double* tot2, cudaStream_t s) {
  launch_k(slab_state_init_kernel, 1, 1, 0, s, st, tot2);
}
void launch_slab_finalize(ImgState* st, const double* tot, int k, double* rre_hist, double* res_hist, int track,
                          int stop_kind, double eps, cudaStream_t s) {
  launch_k(slab_finalize_kernel, 1, 1, 0, s, st, tot, k, rre_hist, res_hist, track, stop_kind, eps);
}
void launch_slab_best_copy(const ImgState* st, const double* x, double* best, size_t n, cudaStream_t s) {
  launch_k(slab_best_copy_kernel, 1184, 256, 0, s, st, x, best, n);
}

void launch_zero(double* p, size_t n, cudaStream_t s) {
  launch_k(zero_kernel, (unsigned)((n + 255) / 256 < 4096 ? (n + 255) / 256 : 4096), 256, 0, s, p, n);
}

}  // namespace dbx
