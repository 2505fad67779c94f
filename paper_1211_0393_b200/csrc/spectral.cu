// spectral.cu — FFT-form kernels of the AR path.
//
// (1) FFT correlation blur (replaces correlate_valid_fft, blur.hpp:56-68, the
//     reference's own engine for q > 7): three passes over a batch,
//       conv_row_fwd : AR-extend each FOV row on the fly (boundary.hpp:56-62),
//                      real FFT of length L2 (two rows packed per complex FFT),
//                      store the Lh = L2/2+1 half spectrum
//       conv_col     : synthesise the vertical AR extension rows in the
//                      spectral domain (FFT is linear: Z[-i] = 2 Z[0] - Z[i]),
//                      FFT L1, multiply by the precomputed kernel spectrum
//                      conj(W^) / (L1 L2), inverse FFT, keep the n1 valid rows
//       conv_row_inv : inverse real FFT, crop, fused epilogue (store /
//                      r = g - A x with ||r||^2 / x += tau*A'r with norms).
// (2) AR transforms T~ / T and the plain DST-I Q (replaces sine1_forward +
//     r2r RODFT00, ar_forward / ar_inverse, tensor_map, transforms.hpp:114-192,
//     and the Hadamard of filter_apply, spectral.hpp:161-165): the DST-I of
//     length N-1 is the imaginary part of two real length-N DFTs, packed into
//     one complex DFT of z_j = v_j (1 + i(-1)^j); that DFT (N = n-1 is never
//     smooth: 255, 511, 1023, 2047, 8191) is a Bluestein chirp-z convolution
//     over a power-of-two M >= 2N-1 in shared memory.
//       dst_rows : one line per row, optional Hadamard by d / axpy + norms
//       dst_cols : CW adjacent columns per CTA (32-byte row segments); runs
//                  T~, multiplies by the d column, runs T — the whole column
//                  half of D = T diag(d) T~ in one pass.
#include <cuda_runtime.h>

#include "dbx_internal.h"
#include "fft.cuh"
#include "spectral.h"

namespace dbx {

using fft::cadd;
using fft::cmul;
using fft::csub;
using fft::pad;
using fft::padded_len;

namespace {

// threads per FFT line: conv lines get one radix-8 butterfly per thread, DST
// lines (power-of-two M) two; both capped at 256 so a CTA of <= 512 threads
// keeps >= 128 registers per thread for the in-register radix stages.
__host__ __device__ constexpr int line_threads(int L, int per) {
  if (L & 1) {
    // direct odd length: the first (largest-prime) stage runs packed across
    // the CTA's lines, so size the line for the second stage's butterflies
    // (1023 = 31*11*3 -> 93 radix-11 butterflies -> 96 threads)
    const int r1 = fft::next_radix(L);
    const int r2 = fft::next_radix(L / r1);
    int t = ((r2 ? L / r2 : L) + 31) / 32 * 32;
    return t < 32 ? 32 : (t > 256 ? 256 : t);
  }
  int t = (L / per + 31) / 32 * 32;
  return t < 32 ? 32 : (t > 256 ? 256 : t);
}
// lines (rows / columns / row pairs) per CTA for a line length L
__host__ __device__ constexpr int lines_for(int L, int budget_bytes, int per) {
  const int bytes = padded_len(L) * 16;
  int g = budget_bytes / bytes;
  g = g < 1 ? 1 : (g > 4 ? 4 : g);
  // odd lengths carry radix <= 31 butterflies in registers: cap the CTA at 256
  // threads so each thread may use up to 255 registers without spilling
  // odd lengths: radix <= 31 butterflies (~170 registers) -> at most 192
  // threads so two CTAs share an SM; even lengths: 384 (2 CTAs/SM at <= 85 regs)
  const int cap = (L & 1) ? 192 : 384;
  while (g > 1 && g * line_threads(L, per) > cap) --g;
  return g;
}
// DST lines: direct odd-length DFTs (radix up to 31) get one butterfly-sized
// share per thread (L/8), power-of-two Bluestein lines two radix-8 butterflies.
__host__ __device__ constexpr int dst_per(int L) { return (L & 1) ? 8 : 16; }
constexpr int kConvBudget = 100 * 1024;
constexpr int kDstBudget = 160 * 1024;

// Asynchronous global -> shared copies (LDGSTS): operands needed only after a
// transform are staged at kernel start without holding registers.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait_group() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory"); }

// Bulk L2 prefetch of a contiguous row (TMA unit; no registers, no smem).
__device__ __forceinline__ void prefetch_l2(const void* p, unsigned bytes) {
  const unsigned long long a = (unsigned long long)p;
  if ((a & 15) || (bytes & 15) || bytes == 0) return;
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;\n" ::"l"(p), "r"(bytes) : "memory");
}

// Twiddle table of an FFT length L staged into shared memory (cp.async group
// committed here) when `smem_ok`, else read from global (L1/L2).
template <int L, bool SMEM>
__device__ __forceinline__ const double2* stage_twiddles(double2* dst, const double2* src) {
  if constexpr (SMEM) {
    for (int i = threadIdx.x; i < L; i += blockDim.x) cp_async16(dst + i, src + i);
    cp_async_commit();
    return dst;
  } else {
    cp_async_commit();  // keep group numbering uniform
    return src;
  }
}
constexpr int kSmemCap = 200 * 1024;

__device__ __forceinline__ double hext(const double* __restrict__ x, int i, int j, int n2) {
  const double* row = x + (size_t)i * n2;
  if (j < 0) return 2.0 * row[0] - row[-j];
  if (j >= n2) return 2.0 * row[n2 - 1] - row[2 * (n2 - 1) - j];
  return row[j];
}

template <int NT>
__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < NT / 32; ++i) s += red[i];
  return s;
}

// Shared epilogue of the passes that produce final image values.
struct Epi {
  int mode;  // EPI_STORE / EPI_RESID / EPI_AXPY / EPI_HADAMARD
  double* y;
  const double* g;
  const double* xo;
  const double* f;
  const double* d;
  double tau;
  double p0 = 0.0, p1 = 0.0;
  __device__ __forceinline__ void put(size_t o, double v) {
    if (mode == SPEC_STORE) {
      y[o] = v;
    } else if (mode == SPEC_HADAMARD) {
      y[o] = v * d[o];
    } else if (mode == SPEC_RESID) {
      const double rv = g[o] - v;
      y[o] = rv;
      p0 += rv * rv;
    } else {
      const double xv = xo[o] + tau * v;
      y[o] = xv;
      p0 += xv * xv;
      if (f) {
        const double e = xv - f[o];
        p1 += e * e;
      }
    }
  }
  // Same with the operands already in registers: pa = x_{k-1} / g / d, pb = f.
  __device__ __forceinline__ void put_pre(size_t o, double v, double pa, double pb) {
    if (mode == SPEC_STORE) {
      y[o] = v;
    } else if (mode == SPEC_HADAMARD) {
      y[o] = v * pa;
    } else if (mode == SPEC_RESID) {
      const double rv = pa - v;
      y[o] = rv;
      p0 += rv * rv;
    } else {
      const double xv = pa + tau * v;
      y[o] = xv;
      p0 += xv * xv;
      if (f) {
        const double e = xv - pb;
        p1 += e * e;
      }
    }
  }
};

template <int NT>
__device__ __forceinline__ void write_partials(const SpecArgs& a, Epi& e, double* red, int b) {
  if (!(a.epi == SPEC_RESID || a.epi == SPEC_AXPY) || !a.part.p) return;
  const int cta = blockIdx.x;
  double* P = a.part.p + (size_t)b * NUM_SLOTS * a.part.cap;
  const double s0 = block_sum<NT>(e.p0, red);
  if (a.epi == SPEC_RESID) {
    if (threadIdx.x == 0) P[SLOT_R2 * a.part.cap + cta] = s0;
  } else {
    if (threadIdx.x == 0) P[SLOT_X2 * a.part.cap + cta] = s0;
    const double s1 = block_sum<NT>(e.p1, red);
    if (threadIdx.x == 0) P[SLOT_XF2 * a.part.cap + cta] = s1;
  }
}

__device__ __forceinline__ Epi make_epi(const SpecArgs& a, int b, size_t N) {
  Epi e;
  e.mode = a.epi;
  e.y = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N));
  e.g = a.g ? a.g + (size_t)b * N : nullptr;
  e.xo = a.epi == SPEC_AXPY ? resolve_ptr(a.xold, a.st, a.xoldsel, b, a.batch, N) : nullptr;
  e.f = (a.epi == SPEC_AXPY && a.f) ? a.f + (size_t)b * N : nullptr;
  e.d = a.d;
  e.tau = a.tau;
  return e;
}

// ---------------------------------------------------------------------------
// FFT correlation
// ---------------------------------------------------------------------------
// Shared-memory plan of a conv kernel: G line buffers, optionally the twiddle
// table (TW) and, for conv_col, the G kernel-spectrum columns (HS).
template <int L, int G>
struct ConvSmem {
  static constexpr int lines = G * padded_len(L);
  static constexpr bool HS = (2 * lines) * 16 <= kSmemCap;          // conv_col H staging
  static constexpr bool TW = (lines + (HS ? lines : 0) + L) * 16 <= kSmemCap;
  static constexpr bool TW_ROW = (lines + L) * 16 <= kSmemCap;      // row kernels
  static constexpr size_t col_bytes = (size_t)(lines + (HS ? lines : 0) + (TW ? L : 0)) * 16;
  static constexpr size_t row_bytes = (size_t)(lines + (TW_ROW ? L : 0)) * 16;
};

template <int L2>
__global__ void __launch_bounds__(lines_for(L2, kConvBudget, 8) * line_threads(L2, 8))
conv_row_fwd(SpecArgs a) {
  constexpr int T = line_threads(L2, 8), G = lines_for(L2, kConvBudget, 8);
  using SM = ConvSmem<L2, G>;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  const int g = threadIdx.x / T, t = threadIdx.x - g * T;
  double2* buf = sm + g * padded_len(L2);
  const double2* tw = stage_twiddles<L2, SM::TW_ROW>(sm + SM::lines, a.conv.tw2);
  const int n1 = a.n1, n2 = a.n2, q2 = a.q2, Lh = a.conv.Lh;
  const size_t N = (size_t)n1 * n2;
  const double* x = resolve_ptr(a.in, a.st, a.insel, b, a.batch, N);
  const int ra = (blockIdx.x * G + g) * 2, rb = ra + 1;
  const int wext = n2 + 2 * q2;
  // all of this thread's loads are issued before any smem store (one DRAM
  // round trip per kernel instead of one per element)
  constexpr int PF = (L2 + T - 1) / T;
  double va[PF], vb[PF];
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int p = t + i * T;
    va[i] = 0.0;
    vb[i] = 0.0;
    if (p < wext) {
      const int j = p - q2;
      if (ra < n1) va[i] = hext(x, ra, j, n2);
      if (rb < n1) vb[i] = hext(x, rb, j, n2);
    }
  }
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int p = t + i * T;
    if (p < L2) buf[pad<L2>(p)] = make_double2(va[i], vb[i]);
  }
  cp_async_wait_all();
  __syncthreads();
  fft::fft<L2, -1, T>(buf, tw, t);
  double2* Z = a.zbuf + (size_t)b * n1 * Lh;
  for (int k = t; k < Lh; k += T) {
    const double2 zk = buf[pad<L2>(k)], zm = buf[pad<L2>(k == 0 ? 0 : L2 - k)];
    if (ra < n1) Z[(size_t)ra * Lh + k] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    if (rb < n1) Z[(size_t)rb * Lh + k] = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
  }
}

template <int L1>
__global__ void __launch_bounds__(lines_for(L1, kConvBudget, 8) * line_threads(L1, 8))
conv_col(SpecArgs a) {
  constexpr int T = line_threads(L1, 8), G = lines_for(L1, kConvBudget, 8);
  constexpr int NT = T * G;
  using SM = ConvSmem<L1, G>;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  const int g = threadIdx.x / T, t = threadIdx.x - g * T;
  const int n1 = a.n1, q1 = a.q1, Lh = a.conv.Lh;
  const int k0 = blockIdx.x * G;
  const int kk = k0 + g;
  // group 0: twiddles; group 1: this CTA's kernel-spectrum columns ([k2][k1]
  // layout, contiguous in p) -- both land while the columns are loaded / FFT'd
  double2* hst = sm + SM::lines + g * padded_len(L1);
  const double2* tw = stage_twiddles<L1, SM::TW>(sm + SM::lines + (SM::HS ? SM::lines : 0), a.conv.tw1);
  const double2* Hcol = a.conv.H + (size_t)(kk < Lh ? kk : 0) * L1;
  if constexpr (SM::HS) {
    for (int p = t; p < L1; p += T) cp_async16(hst + p, Hcol + p);
  }
  cp_async_commit();
  const double2* Z = a.zbuf + (size_t)b * n1 * Lh;
  const int hext_rows = n1 + 2 * q1;
  // load the G columns with the vertical AR extension synthesised spectrally
  // (loads batched in registers first, then stored)
  constexpr int PF = (L1 * G + NT - 1) / NT;
  double2 v[PF];
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int idx = threadIdx.x + i * NT;
    const int p = idx / G, gg = idx - p * G, k = k0 + gg;
    v[i] = make_double2(0.0, 0.0);
    if (idx < L1 * G && k < Lh && p < hext_rows) {
      const int rho = p - q1;
      if (rho < 0) {
        const double2 z0 = Z[k], zi = Z[(size_t)(-rho) * Lh + k];
        v[i] = make_double2(2.0 * z0.x - zi.x, 2.0 * z0.y - zi.y);
      } else if (rho >= n1) {
        const double2 z0 = Z[(size_t)(n1 - 1) * Lh + k], zi = Z[(size_t)(2 * (n1 - 1) - rho) * Lh + k];
        v[i] = make_double2(2.0 * z0.x - zi.x, 2.0 * z0.y - zi.y);
      } else {
        v[i] = Z[(size_t)rho * Lh + k];
      }
    }
  }
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int idx = threadIdx.x + i * NT;
    const int p = idx / G, gg = idx - p * G;
    if (idx < L1 * G) sm[gg * padded_len(L1) + pad<L1>(p)] = v[i];
  }
  cp_async_wait_group<1>();  // twiddles landed (H may still be in flight)
  __syncthreads();
  double2* buf = sm + g * padded_len(L1);
  fft::fft<L1, -1, T>(buf, tw, t);
  cp_async_wait_all();  // each thread multiplies only the entries it staged
  if constexpr (SM::HS) {
    for (int p = t; p < L1; p += T) buf[pad<L1>(p)] = cmul(buf[pad<L1>(p)], hst[p]);
  } else {
    for (int p = t; p < L1; p += T) buf[pad<L1>(p)] = cmul(buf[pad<L1>(p)], __ldg(Hcol + p));
  }
  __syncthreads();
  fft::fft<L1, +1, T>(buf, tw, t);
  double2* Y = a.ybuf + (size_t)b * n1 * Lh;
  for (int idx = threadIdx.x; idx < n1 * G; idx += NT) {
    const int p = idx / G, gg = idx - p * G, k = k0 + gg;
    if (k < Lh) Y[(size_t)p * Lh + k] = sm[gg * padded_len(L1) + pad<L1>(p)];
  }
}

template <int L2>
__global__ void __launch_bounds__(lines_for(L2, kConvBudget, 8) * line_threads(L2, 8))
conv_row_inv(SpecArgs a) {
  constexpr int T = line_threads(L2, 8), G = lines_for(L2, kConvBudget, 8);
  constexpr int NT = T * G;
  using SM = ConvSmem<L2, G>;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double red[32];
  const int g = threadIdx.x / T, t = threadIdx.x - g * T;
  double2* buf = sm + g * padded_len(L2);
  const double2* tw = stage_twiddles<L2, SM::TW_ROW>(sm + SM::lines, a.conv.tw2);
  const int n1 = a.n1, n2 = a.n2, Lh = a.conv.Lh;
  const size_t N = (size_t)n1 * n2;
  const int ra = (blockIdx.x * G + g) * 2, rb = ra + 1;
  Epi e = make_epi(a, b, N);
  // bulk-prefetch this pair's epilogue operand rows into L2 while the
  // inverse FFT runs (no registers, no shared memory)
  if (t == 0) {
    const unsigned bytes = (unsigned)(n2 * sizeof(double));
    for (int rr = ra; rr <= rb && rr < n1; ++rr) {
      const size_t o = (size_t)rr * n2;
      if (e.mode == SPEC_RESID) prefetch_l2(e.g + o, bytes);
      if (e.mode == SPEC_AXPY) {
        prefetch_l2(e.xo + o, bytes);
        if (e.f) prefetch_l2(e.f + o, bytes);
      }
    }
  }
  const double2* Y = a.ybuf + (size_t)b * n1 * Lh;
  // only the Lh stored spectra are read (the upper half is their conjugate);
  // loads batched in registers before the smem stores
  constexpr int PF = (L2 / 2 + 1 + T - 1) / T;
  double2 A[PF], Bv[PF];
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int k = t + i * T;
    A[i] = make_double2(0.0, 0.0);
    Bv[i] = A[i];
    if (k < Lh) {
      if (ra < n1) A[i] = Y[(size_t)ra * Lh + k];
      if (rb < n1) Bv[i] = Y[(size_t)rb * Lh + k];
    }
  }
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int k = t + i * T;
    if (k < Lh) {
      // Z_k = A_k + i B_k and Z_{L2-k} = conj(A_k) + i conj(B_k)
      buf[pad<L2>(k)] = make_double2(A[i].x - Bv[i].y, A[i].y + Bv[i].x);
      if (k > 0 && k < L2 - k) buf[pad<L2>(L2 - k)] = make_double2(A[i].x + Bv[i].y, Bv[i].x - A[i].y);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  fft::fft<L2, +1, T>(buf, tw, t);
  for (int c = t; c < n2; c += T) {
    const double2 v = buf[pad<L2>(c)];
    if (ra < n1) e.put((size_t)ra * n2 + c, v.x);
    if (rb < n1) e.put((size_t)rb * n2 + c, v.y);
  }
  write_partials<NT>(a, e, red, b);
}

// ---------------------------------------------------------------------------
// Bluestein DST-I / AR transforms
// ---------------------------------------------------------------------------
// Fill one padded line with a_j = z_j w_j, z_j = v_j (1 + i(-1)^j), j in [1, N).
// `val(j)` returns v_j (1-based interior index).
// Two forms of the N-point DFT of z: BLUE = Bluestein chirp-z over a power of
// two L = M >= 2N-1 (any N); !BLUE = direct mixed-radix FFT of length L = N
// (N with prime factors <= 31, e.g. 255 = 3.5.17, 1023 = 3.11.31).
template <bool BLUE>
__device__ __forceinline__ double2 pre(double2 z, const BlueTables& bt, int j) {
  if constexpr (BLUE) return cmul(z, __ldg(bt.chirp + j));
  else return z;
}

template <int M, int T, bool BLUE, typename F>
__device__ __forceinline__ void blue_fill(double2* buf, const BlueTables& bt, int t, F val) {
  const int N = bt.N;
  // every load of the thread (line values, chirp) is issued before any store
  constexpr int PF = (M + T - 1) / T;
  double2 v[PF];
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int j = t + i * T;
    v[i] = make_double2(0.0, 0.0);
    if (j >= 1 && j < N) {
      const double z = val(j);
      v[i] = pre<BLUE>(make_double2(z, (j & 1) ? -z : z), bt, j);
    }
  }
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int j = t + i * T;
    if (j < M) buf[pad<M>(j)] = v[i];
  }
}

// BLUE: FFT, multiply by the kernel spectrum, inverse FFT.  Direct: one FFT.
// Shared-memory plan of a DST kernel: G line buffers, G x 2 real staging rows
// (epilogue operands / d column and T~ output), then the twiddle table if it
// fits.
template <int L, int G, bool BLUE>
struct DstSmem {
  static constexpr int LMAX = BLUE ? L / 2 + 1 : L + 1;
  static constexpr size_t base = (size_t)G * padded_len(L) * 16 + (size_t)G * 2 * LMAX * 8;
  static constexpr size_t tw_off = (base + 15) / 16 * 16;
  static constexpr bool TW = tw_off + (size_t)L * 16 <= kSmemCap;
  static constexpr size_t bytes = TW ? tw_off + (size_t)L * 16 : base;
};

template <int M, int T, int G, bool BLUE>
__device__ __forceinline__ void blue_core(double2* sm, double2* buf, const BlueTables& bt, const double2* tw,
                                          int t) {
  cp_async_wait_group<1>();  // the twiddle group (committed first) has landed
  __syncthreads();
  if constexpr (!BLUE) {
    // direct odd length: large-prime stages packed across the CTA's G lines
    fft::fft_cta<M, -1, T, G>(sm, tw, threadIdx.x);
    return;
  }
  fft::fft<M, -1, T>(buf, tw, t);
  if constexpr (BLUE) {
    for (int j = t; j < M; j += T) buf[pad<M>(j)] = cmul(buf[pad<M>(j)], __ldg(bt.bhat + j));
    __syncthreads();
    fft::fft<M, +1, T>(buf, tw, t);
  }
}

// DST-I output y_k (k in [1, N)) from Z = DFT_N(z) (post-chirp applied here
// for BLUE), scaled by sqrt(2/N): Q v = sqrt(2/N) sum_j v_j sin(pi j k / N).
// Even k = 2l: -Im DFT(v)_l; odd k: -Im DFT((-1)^j v)_{(k+N)/2} (N odd).
template <int M, bool BLUE>
__device__ __forceinline__ double blue_out(const double2* buf, const BlueTables& bt, int k) {
  const int N = bt.N;
  const int l = (k & 1) == 0 ? (k >> 1) : ((k + N) >> 1);
  const double2 zl = pre<BLUE>(buf[pad<M>(l)], bt, l);
  const double2 zm = pre<BLUE>(buf[pad<M>(N - l)], bt, N - l);
  return (k & 1) == 0 ? 0.5 * bt.scale * (zm.y - zl.y) : 0.5 * bt.scale * (zl.x - zm.x);
}

// Row pass: one AR (or SineI) transform per row, fused epilogue.
template <int M, bool BLUE>
__global__ void __launch_bounds__(lines_for(M, kDstBudget, dst_per(M)) * line_threads(M, dst_per(M)), (M & 1) ? 2 : 1)
dst_rows(SpecArgs a) {
  constexpr int T = line_threads(M, dst_per(M)), G = lines_for(M, kDstBudget, dst_per(M));
  constexpr int NT = T * G;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double red[32];
  const int g = threadIdx.x / T, t = threadIdx.x - g * T;
  double2* buf = sm + g * padded_len(M);
  const int n1 = a.n1, n = a.n2;
  const size_t N = (size_t)n1 * n;
  const BlueTables& bt = a.blue2;
  using SMP = DstSmem<M, G, BLUE>;
  const double2* tw = stage_twiddles<M, SMP::TW>(
      reinterpret_cast<double2*>(reinterpret_cast<char*>(sm) + SMP::tw_off), bt.tw);
  const int r = blockIdx.x * G + g;
  const bool live = r < n1;
  const double* in = resolve_ptr(a.in, a.st, a.insel, b, a.batch, N) + (size_t)(live ? r : 0) * n;
  const int kind = a.kind1;
  const double v0 = in[0], ve = in[n - 1];
  const double* p = bt.p;
  if (kind == DBX_KIND_SINEI) {
    blue_fill<M, T, BLUE>(buf, bt, t, [&](int j) { return live ? in[j - 1] : 0.0; });
  } else if (kind == DBX_KIND_ARINV) {
    blue_fill<M, T, BLUE>(buf, bt, t, [&](int j) {
      return live ? (in[j] - v0 * __ldg(p + j - 1)) - ve * __ldg(p + n - 2 - j) : 0.0;
    });
  } else {
    blue_fill<M, T, BLUE>(buf, bt, t, [&](int j) { return live ? in[j] : 0.0; });
  }
  // Stage the epilogue operands (x_{k-1} and f, or g, or d) into shared
  // memory with cp.async at kernel start: their HBM latency hides behind the
  // transform and they cost no registers.  A line holds at most M/2+1
  // (Bluestein) or M+1 (direct) pixels.
  constexpr int LMAX = BLUE ? M / 2 + 1 : M + 1;
  double* stA = reinterpret_cast<double*>(sm + G * padded_len(M)) + g * 2 * LMAX;
  double* stB = stA + LMAX;
  Epi e = make_epi(a, b, N);
  const size_t ro = (size_t)(live ? r : 0) * n;
  if (live && e.mode != SPEC_STORE) {
    const double* srcA = e.mode == SPEC_AXPY ? e.xo : e.mode == SPEC_RESID ? e.g : e.d;
    for (int k = t; k < n; k += T) {
      cp_async8(stA + k, srcA + ro + k);
      if (e.mode == SPEC_AXPY && e.f) cp_async8(stB + k, e.f + ro + k);
    }
  }
  cp_async_commit();
  blue_core<M, T, G, BLUE>(sm, buf, bt, tw, t);
  cp_async_wait_all();  // each thread reads back only what it staged
  if (live) {
    const double al = bt.alpha, ia = 1.0 / bt.alpha;
    const double a0 = ia * v0, a1 = ia * ve;
    for (int k = t; k < n; k += T) {
      double v;
      if (kind == DBX_KIND_SINEI) {
        v = blue_out<M, BLUE>(buf, bt, k + 1);
      } else if (kind == DBX_KIND_ARINV) {
        v = (k == 0) ? al * v0 : (k == n - 1) ? al * ve : blue_out<M, BLUE>(buf, bt, k);
      } else if (k == 0) {
        v = a0;
      } else if (k == n - 1) {
        v = a1;
      } else {
        v = blue_out<M, BLUE>(buf, bt, k);
        v += a0 * __ldg(p + k - 1);
        v += a1 * __ldg(p + n - 2 - k);
      }
      e.put_pre(ro + k, v, stA[k], stB[k]);
    }
  }
  write_partials<NT>(a, e, red, b);
}

// Column pass: CW adjacent columns per CTA; kind1, then optional Hadamard by
// the d column, then optional kind2 (-1 = none).  Output with STORE epilogue.
template <int M, bool BLUE>
__global__ void __launch_bounds__(lines_for(M, kDstBudget, dst_per(M)) * line_threads(M, dst_per(M)), (M & 1) ? 2 : 1)
dst_cols(SpecArgs a) {
  constexpr int T = line_threads(M, dst_per(M)), G = lines_for(M, kDstBudget, dst_per(M));
  constexpr int NT = T * G;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double vb0[4], vbe[4];
  const int g = threadIdx.x / T, t = threadIdx.x - g * T;
  double2* buf = sm + g * padded_len(M);
  const int n = a.n1, n2 = a.n2;
  const size_t N = (size_t)n * n2;
  const BlueTables& bt = a.blue1;
  using SMP = DstSmem<M, G, BLUE>;
  const double2* tw = stage_twiddles<M, SMP::TW>(
      reinterpret_cast<double2*>(reinterpret_cast<char*>(sm) + SMP::tw_off), bt.tw);
  const int c0 = blockIdx.x * G;
  const int c = c0 + g;
  const bool live = c < n2;
  const double* in = resolve_ptr(a.in, a.st, a.insel, b, a.batch, N);
  const double* p = bt.p;
  const int NL = bt.N;

  // staging areas after the G line buffers: d column and T~ output (real)
  constexpr int LMAX = BLUE ? M / 2 + 1 : M + 1;
  double* dst_d = reinterpret_cast<double*>(sm + G * padded_len(M)) + g * 2 * LMAX;
  double* midS = dst_d + LMAX;
  if (a.kind2 >= 0 && a.d) {
    for (int idx = threadIdx.x; idx < n * G; idx += NT) {
      const int j = idx / G, gg = idx - j * G, cc = c0 + gg;
      if (cc < n2)
        cp_async8(reinterpret_cast<double*>(sm + G * padded_len(M)) + gg * 2 * LMAX + j, a.d + (size_t)j * n2 + cc);
    }
  }
  cp_async_commit();

  // ---- first transform (input from global, column-strided, 32 B segments) ----
  if (threadIdx.x < G) {
    const int cc = c0 + threadIdx.x;
    vb0[threadIdx.x] = cc < n2 ? in[cc] : 0.0;
    vbe[threadIdx.x] = cc < n2 ? in[(size_t)(n - 1) * n2 + cc] : 0.0;
  }
  __syncthreads();
  const int kind1 = a.kind1, kind2 = a.kind2;
  {
    constexpr int PF = (M * G + NT - 1) / NT;
    double2 v[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) {
      const int idx = threadIdx.x + i * NT;
      const int j = idx / G, gg = idx - j * G, cc = c0 + gg;
      v[i] = make_double2(0.0, 0.0);
      if (idx < M * G && j >= 1 && j < NL && cc < n2) {
        double z;
        if (kind1 == DBX_KIND_SINEI) z = in[(size_t)(j - 1) * n2 + cc];
        else if (kind1 == DBX_KIND_ARINV)
          z = (in[(size_t)j * n2 + cc] - vb0[gg] * __ldg(p + j - 1)) - vbe[gg] * __ldg(p + n - 2 - j);
        else z = in[(size_t)j * n2 + cc];
        v[i] = pre<BLUE>(make_double2(z, (j & 1) ? -z : z), bt, j);
      }
    }
#pragma unroll
    for (int i = 0; i < PF; ++i) {
      const int idx = threadIdx.x + i * NT;
      const int j = idx / G, gg = idx - j * G;
      if (idx < M * G) sm[gg * padded_len(M) + pad<M>(j)] = v[i];
    }
  }
  blue_core<M, T, G, BLUE>(sm, buf, bt, tw, t);

  double* out = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N));
  if (kind2 < 0) {
    // single transform: write the column directly
    __syncthreads();
    for (int idx = threadIdx.x; idx < n * G; idx += NT) {
      const int k = idx / G, gg = idx - k * G, cc = c0 + gg;
      if (cc >= n2) continue;
      const double2* bb = sm + gg * padded_len(M);
      double v;
      if (kind1 == DBX_KIND_SINEI) v = blue_out<M, BLUE>(bb, bt, k + 1);
      else if (kind1 == DBX_KIND_ARINV) v = (k == 0) ? bt.alpha * vb0[gg] : (k == n - 1) ? bt.alpha * vbe[gg] : blue_out<M, BLUE>(bb, bt, k);
      else {
        const double ia = 1.0 / bt.alpha, a0 = ia * vb0[gg], a1 = ia * vbe[gg];
        if (k == 0) v = a0;
        else if (k == n - 1) v = a1;
        else {
          v = blue_out<M, BLUE>(bb, bt, k);
          v += a0 * __ldg(p + k - 1);
          v += a1 * __ldg(p + n - 2 - k);
        }
      }
      if (a.epi == SPEC_HADAMARD) v *= a.d[(size_t)k * n2 + cc];
      out[(size_t)k * n2 + cc] = v;
    }
    return;
  }

  // ---- middle: u = T~ result (AR inverse), v' = u o d, refill for kind2 = T ----
  // (the d column was staged into shared memory by cp.async at kernel start)
  cp_async_wait_all();
  __syncthreads();
  for (int j = t; j < M; j += T) {  // interior index 1..NL-1
    double m = 0.0;
    if (live && j >= 1 && j < NL) {
      const double u = blue_out<M, BLUE>(buf, bt, j);
      m = a.d ? u * dst_d[j] : u;
    }
    if (j < LMAX) midS[j] = m;
  }
  __syncthreads();
  if (threadIdx.x < G) {
    const int cc = c0 + threadIdx.x;
    double u0 = bt.alpha * vb0[threadIdx.x], ue = bt.alpha * vbe[threadIdx.x];
    if (a.d && cc < n2) {
      u0 *= a.d[cc];
      ue *= a.d[(size_t)(n - 1) * n2 + cc];
    }
    vb0[threadIdx.x] = u0;
    vbe[threadIdx.x] = ue;
  }
  for (int j = t; j < M; j += T) {
    double2 v = make_double2(0.0, 0.0);
    if (j >= 1 && j < NL) {
      const double m = midS[j];
      v = pre<BLUE>(make_double2(m, (j & 1) ? -m : m), bt, j);
    }
    buf[pad<M>(j)] = v;
  }
  blue_core<M, T, G, BLUE>(sm, buf, bt, tw, t);
  // ---- T (AR forward) output, coalesced 32 B row segments ----
  const double ia = 1.0 / bt.alpha;
  for (int idx = threadIdx.x; idx < n * G; idx += NT) {
    const int k = idx / G, gg = idx - k * G, cc = c0 + gg;
    if (cc >= n2) continue;
    const double2* bb = sm + gg * padded_len(M);
    const double a0 = ia * vb0[gg], a1 = ia * vbe[gg];
    double v;
    if (k == 0) v = a0;
    else if (k == n - 1) v = a1;
    else {
      v = blue_out<M, BLUE>(bb, bt, k);
      v += a0 * __ldg(p + k - 1);
      v += a1 * __ldg(p + n - 2 - k);
    }
    out[(size_t)k * n2 + cc] = v;
  }
}

template <typename K>
bool set_smem(K kernel, size_t bytes) {
  if (bytes > 227 * 1024) return false;
  if (bytes > 48 * 1024)
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess;
  return true;
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers (size dispatch)
// ---------------------------------------------------------------------------
#define DBX_CONV_LIST(X)                                                                       \
  X(64) X(72) X(80) X(96) X(128) X(144) X(160) X(192) X(256) X(270) X(288) X(320) X(384) X(512) \
  X(540) X(576) X(640) X(768) X(1024) X(1080) X(1152) X(1280) X(1536) X(2048) X(2160) X(2304) \
  X(2560) X(3072) X(4096) X(4320) X(4608) X(5120) X(6144) X(8192) X(8640)
#define DBX_BLUE_LIST(X) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192)

int conv_supported_len(int need) {
  int best = 0;
#define X(L) if (best == 0 && (L) >= need) best = (L);
  DBX_CONV_LIST(X)
#undef X
  return best;
}

int blue_supported_len(int need) {
  int best = 0;
#define X(L) if (best == 0 && (L) >= need) best = (L);
  DBX_BLUE_LIST(X)
#undef X
  return best;
}

int launch_conv_row_fwd(const SpecArgs& a, cudaStream_t s) {
  const int L2 = a.conv.L2;
#define X(L)                                                                             \
  if (L2 == (L)) {                                                                       \
    constexpr int T = line_threads(L, 8), G = lines_for(L, kConvBudget, 8);                     \
    const size_t sm = ConvSmem<L, G>::row_bytes;                                         \
    static bool init = false;                                                            \
    if (!init) { if (!set_smem(conv_row_fwd<L>, sm)) return -1; init = true; }                            \
    dim3 grid((a.n1 + 2 * G - 1) / (2 * G), a.batch);                                    \
    conv_row_fwd<L><<<grid, T * G, sm, s>>>(a);                                          \
    return (int)grid.x;                                                                  \
  }
  DBX_CONV_LIST(X)
#undef X
  return -1;
}

int launch_conv_col(const SpecArgs& a, cudaStream_t s) {
  const int L1 = a.conv.L1;
#define X(L)                                                                             \
  if (L1 == (L)) {                                                                       \
    constexpr int T = line_threads(L, 8), G = lines_for(L, kConvBudget, 8);                     \
    const size_t sm = ConvSmem<L, G>::col_bytes;                                         \
    static bool init = false;                                                            \
    if (!init) { if (!set_smem(conv_col<L>, sm)) return -1; init = true; }                                \
    dim3 grid((a.conv.Lh + G - 1) / G, a.batch);                                         \
    conv_col<L><<<grid, T * G, sm, s>>>(a);                                              \
    return (int)grid.x;                                                                  \
  }
  DBX_CONV_LIST(X)
#undef X
  return -1;
}

int launch_conv_row_inv(const SpecArgs& a, cudaStream_t s) {
  const int L2 = a.conv.L2;
#define X(L)                                                                             \
  if (L2 == (L)) {                                                                       \
    constexpr int T = line_threads(L, 8), G = lines_for(L, kConvBudget, 8);                     \
    const size_t sm = ConvSmem<L, G>::row_bytes;                                         \
    static bool init = false;                                                            \
    if (!init) { if (!set_smem(conv_row_inv<L>, sm)) return -1; init = true; }                            \
    dim3 grid((a.n1 + 2 * G - 1) / (2 * G), a.batch);                                    \
    conv_row_inv<L><<<grid, T * G, sm, s>>>(a);                                          \
    return (int)grid.x;                                                                  \
  }
  DBX_CONV_LIST(X)
#undef X
  return -1;
}

// DST launch over both forms: BLUE lines use M (power of two), direct lines
// use M == N (odd, prime factors <= 31).
#define DBX_DIRECT_LIST(X) X(15) X(31) X(63) X(255) X(1023) X(4095)

template <int L, bool BLUE>
int dst_rows_launch(const SpecArgs& a, cudaStream_t s) {
  constexpr int T = line_threads(L, dst_per(L)), G = lines_for(L, kDstBudget, dst_per(L));
  const size_t sm = DstSmem<L, G, BLUE>::bytes;
  static bool init = false;
  if (!init) { if (!set_smem(dst_rows<L, BLUE>, sm)) return -1; init = true; }
  dim3 grid((a.n1 + G - 1) / G, a.batch);
  dst_rows<L, BLUE><<<grid, T * G, sm, s>>>(a);
  return (int)grid.x;
}

template <int L, bool BLUE>
int dst_cols_launch(const SpecArgs& a, cudaStream_t s) {
  constexpr int T = line_threads(L, dst_per(L)), G = lines_for(L, kDstBudget, dst_per(L));
  const size_t sm = DstSmem<L, G, BLUE>::bytes;
  static bool init = false;
  if (!init) { if (!set_smem(dst_cols<L, BLUE>, sm)) return -1; init = true; }
  dim3 grid((a.n2 + G - 1) / G, a.batch);
  dst_cols<L, BLUE><<<grid, T * G, sm, s>>>(a);
  return (int)grid.x;
}

int direct_supported_len(int N) {
#define X(L) if (N == (L)) return (L);
  DBX_DIRECT_LIST(X)
#undef X
  return 0;
}

int launch_dst_rows(const SpecArgs& a, cudaStream_t s) {
  const int M = a.blue2.M;
  if (M == a.blue2.N) {
#define X(L) if (M == (L)) return dst_rows_launch<L, false>(a, s);
    DBX_DIRECT_LIST(X)
#undef X
    return -1;
  }
#define X(L) if (M == (L)) return dst_rows_launch<L, true>(a, s);
  DBX_BLUE_LIST(X)
#undef X
  return -1;
}

int launch_dst_cols(const SpecArgs& a, cudaStream_t s) {
  const int M = a.blue1.M;
  if (M == a.blue1.N) {
#define X(L) if (M == (L)) return dst_cols_launch<L, false>(a, s);
    DBX_DIRECT_LIST(X)
#undef X
    return -1;
  }
#define X(L) if (M == (L)) return dst_cols_launch<L, true>(a, s);
  DBX_BLUE_LIST(X)
#undef X
  return -1;
}

int conv_rows_per_cta(int L2) {
#define X(L) if (L2 == (L)) return 2 * lines_for(L, kConvBudget, 8);
  DBX_CONV_LIST(X)
#undef X
  return 0;
}

}  // namespace dbx
