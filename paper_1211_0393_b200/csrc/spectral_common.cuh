// spectral_common.cuh — device helpers shared by the FFT-form kernels
// (spectral.cu: separate passes; fused.cu: fused row pipelines).
#pragma once

#include <cuda_runtime.h>

#include "dbx_internal.h"
#include "fft.cuh"
#include "spectral.h"
#include "pfa.cuh"

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
#ifndef DBX_BIG_LINE_T
#define DBX_BIG_LINE_T 512
#endif
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
  // one line per CTA at L >= 8000 (C5: 8190 / 8192 / 8640): a wider line keeps
  // more warps resident on the SM
  const int cap = L >= 8000 ? DBX_BIG_LINE_T : 256;
  return t < 32 ? 32 : (t > cap ? cap : t);
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
// Resident CTAs per SM the FFT-form row kernels (conv_row_fwd / conv_row_inv)
// are register-capped for at mid lengths (C4's 2160: 92-94 registers = 2 CTAs
// of 256 threads per SM; at 3: C4 7143 -> 7270 Mpx-it/s, profiles/r03_conv_minb_ab.txt).  0 = no minimum (the one-argument launch bounds: an
// explicit 1 is not neutral, see dst.cu).  A/B knob.
#ifndef DBX_CONV_MINB_MID
#define DBX_CONV_MINB_MID 3
#endif
__host__ __device__ constexpr int conv_row_minb(int L) { return (L >= 1500 && L < 4000) ? DBX_CONV_MINB_MID : 0; }
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

// One 32-byte global store of two adjacent complex values (sm_100 256-bit
// STG): the half spectra of a packed row pair go out as one full sector.
__device__ __forceinline__ void st_pair(double2* p, double2 a, double2 b) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(p), "d"(a.x), "d"(a.y), "d"(b.x), "d"(b.y)
               : "memory");
}

// Number of SMs (for prefetch-ahead distances of one resident wave).
__device__ __forceinline__ int nsm() {
  unsigned r;
  asm("mov.u32 %0, %%nsmid;" : "=r"(r));
  return (int)r;
}

// Twiddle table of an FFT length L staged into shared memory (cp.async group
// committed here) when `smem_ok`, else read from global (L1/L2).
template <int L, bool SMEM, int NEED_ = 0>
__device__ __forceinline__ const double2* stage_twiddles(double2* dst, const double2* src) {
  if constexpr (SMEM) {
    constexpr int NEED = NEED_ > 0 ? NEED_ : dst_twiddles_needed(L);
    for (int i = threadIdx.x; i < NEED; i += blockDim.x) cp_async16(dst + i, src + i);
    cp_async_commit();
    return dst;
  } else {
    cp_async_commit();  // keep group numbering uniform
    return src;
  }
}
constexpr int kSmemCap = 200 * 1024;

__device__ __forceinline__ double hext(const double* __restrict__ x, int i, int j, int n2,
                                       int bc = DBX_BC_ANTIREFLECTIVE) {
  const double* row = x + (size_t)i * n2;
  if (bc == DBX_BC_REFLECTIVE) {  // f_{-k} = f_{k-1}, f_{n-1+k} = f_{n-k} (boundary.hpp:49-55)
    if (j < 0) return row[-j - 1];
    if (j >= n2) return row[2 * n2 - 1 - j];
    return row[j];
  }
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

// Epilogue of one output row (elements o0 + k, k in [t, n) step T) with the
// operand loads (x_{k-1} and f / g / d) issued U deep before the stores: the
// stores would otherwise keep the compiler from hoisting a load above them, one
// L2/HBM round trip per element (C4's T + axpy pass: 102 vs 64 us for the plain
// pass).  val(k) gives the transform output k.
template <int U, typename V>
__device__ __forceinline__ void epi_row(Epi& e, size_t o0, int n, int t, int T, V val) {
  for (int k0 = t; k0 < n; k0 += U * T) {
    double pa[U], pb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * T;
      pa[u] = 0.0;
      pb[u] = 0.0;
      if (k < n) {
        const size_t o = o0 + k;
        if (e.mode == SPEC_AXPY) {
          pa[u] = e.xo[o];
          if (e.f) pb[u] = e.f[o];
        } else if (e.mode == SPEC_RESID) {
          pa[u] = e.g[o];
        } else if (e.mode == SPEC_HADAMARD) {
          pa[u] = e.d[o];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int k = k0 + u * T;
      if (k < n) e.put_pre(o0 + k, val(k), pa[u], pb[u]);
    }
  }
}

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
  e.d = a.d ? a.d + (size_t)b * a.dstride : nullptr;
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
  static constexpr int TWN = fft::twiddles_needed(L);               // staged twiddle prefix
  static constexpr bool TW = (lines + (HS ? lines : 0) + TWN) * 16 <= kSmemCap;
  static constexpr bool TW_ROW = (lines + TWN) * 16 <= kSmemCap;    // row kernels
  static constexpr size_t col_bytes = (size_t)(lines + (HS ? lines : 0) + (TW ? TWN : 0)) * 16;
  static constexpr size_t row_bytes = (size_t)(lines + (TW_ROW ? TWN : 0)) * 16;
};

// ---------------------------------------------------------------------------
// Bluestein DST-I / AR transforms
// ---------------------------------------------------------------------------
// Two forms of the N-point DFT in the fused kernels: BLUE = Bluestein chirp-z
// over a power of two M >= 2N-1 (any N); !BLUE = direct mixed-radix FFT of
// length M = N (N with prime factors <= 31, e.g. 255 = 3.5.17, 1023 = 3.11.31).
// (dst.cu adds the Rader core for prime N.)
template <bool BLUE>
__device__ __forceinline__ double2 pre(double2 z, const BlueTables& bt, int j) {
  if constexpr (BLUE) return cmul(z, __ldg(bt.chirp + j));
  else return z;
}

// BLUE: FFT, multiply by the kernel spectrum, inverse FFT.  Direct: one FFT.
template <int M, int T, int G, bool BLUE>
__device__ __forceinline__ void blue_core(double2* sm, double2* buf, const BlueTables& bt, const double2* tw,
                                          int t, double2* pfa_aux = nullptr) {
  cp_async_wait_group<1>();  // the twiddle group (committed first) has landed
  __syncthreads();
  if constexpr (pfa_len(M)) {
    // prime-factor line (pfa.cuh), per-line named barriers
    const int bar = G > 1 ? 1 + (int)threadIdx.x / T : 0;
    pfa_core<M, T>(buf, bt, tw, t, bar, pfa_aux);
    __syncthreads();
    return;
  } else if constexpr (!BLUE) {
    // direct odd length: large-prime stages packed across the CTA's G lines
    fft::fft_cta<M, -1, T, G>(sm, tw, threadIdx.x);
    return;
  } else {
    const int bar = G > 1 ? 1 + (int)threadIdx.x / T : 0;  // per-line named barrier
#ifndef DBX_FUSED_STOCKHAM_BLUE
    // in-place Cooley-Tukey convolution core (fft.cuh ct_convolve, the Rader
    // core of dst.cu): C2's 1024-point Bluestein lines 3763 -> 4052 Mpx-it/s
    // (profiles/r02_fused_ct_ab.txt); -DDBX_FUSED_STOCKHAM_BLUE restores the two
    // Stockham FFTs.  Needs the CT twiddle prefix inside the staged Stockham one.
    static_assert(fft::ct_twiddles_needed(M) <= fft::twiddles_needed(M), "CT twiddle prefix");
    fft::ct_convolve<M, T>(buf, tw, bt.bct, t, bar, nullptr);
#else
    fft::fft<M, -1, T>(buf, tw, t, bar);
    for (int j = t; j < M; j += T) buf[pad<M>(j)] = cmul(buf[pad<M>(j)], __ldg(bt.bhat + j));
    fft::line_sync(bar, T);
    fft::fft<M, +1, T>(buf, tw, t, bar);
#endif
    __syncthreads();  // the split reads other lines' data only after every line finished
  }
}

// ---------------------------------------------------------------------------
// Packed real DST-I: TWO real lines per complex N-point DFT.
//   y_j = sin(pi j/N) (x_j + x_{N-j}) + (x_j - x_{N-j}) / 2   (j in [1, N), y_0 = 0)
//   Y = DFT_N(y):  X_{2l} = -Im Y_l,  X_1 = Re Y_0 / 2,  X_{2l+1} = X_{2l-1} + Re Y_l
// (X_k = sum_j x_j sin(pi j k / N)).  Two lines a, b share one DFT of
// z = y^a + i y^b and are separated by conjugate symmetry, so the transform
// count is half that of one complex DFT per line; the odd outputs are a
// prefix sum (odd_scan).  Works for any N (odd or even).
// sd(h, j) returns (x^h_j + x^h_{N-j}, x^h_j - x^h_{N-j}) for line h in {0, 1}
// and j in [1, N/2]: each thread forms z_j and z_{N-j} from one set of loads
// (sin(pi (N-j)/N) = sin(pi j/N)).
template <int M, int T, bool BLUE, typename F>
__device__ __forceinline__ void pk_fill(double2* buf, const BlueTables& bt, int t, F sd) {
  const int N = bt.N, H = N / 2;
  // positions no pair covers: 0, and the Bluestein zero padding [N, M)
  if (t == 0) buf[pad<M>(0)] = make_double2(0.0, 0.0);
  if constexpr (BLUE)
    for (int p = N + t; p < M; p += T) buf[pad<M>(p)] = make_double2(0.0, 0.0);
  constexpr int HMAX = (BLUE ? M / 2 + 1 : M) / 2;
  constexpr int PF = (HMAX + T - 1) / T;
  // the thread's sine weights first, all in flight at once (one L1/L2 round
  // trip instead of one per element: the loop's shared-memory stores would
  // otherwise keep the compiler from hoisting the global loads)
  double sw[PF];
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int j = 1 + t + i * T;
    sw[i] = j <= H ? __ldg(bt.sn + j) : 0.0;
  }
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int j = 1 + t + i * T;
    if (j <= H) {
      const double s = sw[i];
      const double2 A = sd(0, j), B = sd(1, j);
      const double2 zj = make_double2(fma(s, A.x, 0.5 * A.y), fma(s, B.x, 0.5 * B.y));
      const double2 zm = make_double2(fma(s, A.x, -0.5 * A.y), fma(s, B.x, -0.5 * B.y));
      if constexpr (pfa_len(M)) {  // Good-Thomas input map (pfa.cuh)
        buf[__ldg(bt.dlog + j)] = zj;
        if (N - j != j) buf[__ldg(bt.dlog + N - j)] = zm;
      } else {
        buf[pad<M>(j)] = pre<BLUE>(zj, bt, j);
        if (N - j != j) buf[pad<M>(N - j)] = pre<BLUE>(zm, bt, N - j);
      }
    }
  }
}

// Separate the two lines' spectra (A_l = (Z_l + conj Z_{N-l}) / 2,
// B_l = (Z_l - conj Z_{N-l}) / 2i) into the DST outputs: even k final (scaled),
// odd k the scan terms (unscaled) — odd_scan completes them.
template <int M, bool BLUE>
__device__ __forceinline__ void pk_split(const double2* buf, const BlueTables& bt, double* oa, double* ob, int t,
                                         int T) {
  const int N = bt.N;
  const double hs = 0.5 * bt.scale;
  for (int l = t; 2 * l <= N - 1; l += T) {
    const int m = l == 0 ? 0 : N - l;
    const double2 zl = pre<BLUE>(buf[pad<M>(l)], bt, l);
    const double2 zm = pre<BLUE>(buf[pad<M>(m)], bt, m);
    if (l >= 1) {
      oa[2 * l] = hs * (zm.y - zl.y);
      ob[2 * l] = hs * (zl.x - zm.x);
    }
    if (2 * l + 1 <= N - 1) {
      const double f = l == 0 ? 0.25 : 0.5;
      oa[2 * l + 1] = f * (zl.x + zm.x);
      ob[2 * l + 1] = f * (zl.y + zm.y);
    }
  }
}

// One warp: inclusive prefix sums of o[1], o[3], ..., o[2 cnt - 1], scaled.
__device__ __forceinline__ void odd_scan(double* o, int cnt, double sc, int lane) {
  double carry = 0.0;
  constexpr int RW = 16;  // rows of 32 in flight (one chunk covers 512 outputs)
  for (int base = 0; base < cnt; base += RW * 32) {
    double v[RW];
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      const int m = base + i * 32 + lane;
      v[i] = m < cnt ? o[2 * m + 1] : 0.0;
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int i = 0; i < RW; ++i) {
        const double y = __shfl_up_sync(0xffffffffu, v[i], d);
        if (lane >= d) v[i] += y;
      }
    }
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      const double tot = __shfl_sync(0xffffffffu, v[i], 31);
      const int m = base + i * 32 + lane;
      if (m < cnt) o[2 * m + 1] = (v[i] + carry) * sc;
      carry += tot;
    }
  }
}

// One warp: unscaled inclusive prefix sums of o[2m + 1], m in [lo, hi), in
// place; returns the range total (every lane).
__device__ __forceinline__ double odd_scan_range(double* o, int lo, int hi, int lane) {
  double carry = 0.0;
  constexpr int RW = 8;
  for (int base = lo; base < hi; base += RW * 32) {
    double v[RW];
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      const int m = base + i * 32 + lane;
      v[i] = m < hi ? o[2 * m + 1] : 0.0;
    }
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
#pragma unroll
      for (int i = 0; i < RW; ++i) {
        const double y = __shfl_up_sync(0xffffffffu, v[i], d);
        if (lane >= d) v[i] += y;
      }
    }
#pragma unroll
    for (int i = 0; i < RW; ++i) {
      const double tot = __shfl_sync(0xffffffffu, v[i], 31);
      const int m = base + i * 32 + lane;
      if (m < hi) o[2 * m + 1] = v[i] + carry;
      carry += tot;
    }
  }
  return carry;
}

// Scans of `nlines` output lines of stride LS (doubles), spread over the warps.
__device__ __forceinline__ void odd_scans(double* o, int LS, int nlines, const BlueTables& bt) {
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int s = w; s < nlines; s += nw) odd_scan(o + (size_t)s * LS, bt.N / 2, bt.scale, lane);
}

// ---------------------------------------------------------------------------
// Scan-friendly output layout of the fused kernels (N <= 1025): X_{2l} at
// o[l]; the odd terms X_{2m+1} at o[EB + (m & 15) * STR + (m >> 4)], so lane L
// of the scanning warp owns the contiguous run m = 16L .. 16L+15 with
// conflict-free accesses (STR odd): 16 sequential adds per lane + one warp
// scan of the lane totals, instead of shuffle scans over every element.
template <int LMAX>
struct PkOut {
  static constexpr int EB = LMAX / 2 + 1;                  // even block
  static constexpr int CNT = LMAX / 2;                     // max odd terms
  static constexpr int STR = ((CNT + 15) / 16) | 1;        // odd row stride >= CNT/16
  static constexpr int STR1 = STR < (CNT + 15) / 16 + 1 ? STR + 2 : STR;
  static constexpr int OL = EB + 16 * STR1;                // doubles per output line
  static_assert(CNT <= 512, "one scanning warp covers 32 x 16 odd terms");
};

template <int LMAX>
__device__ __forceinline__ double pk_at(const double* o, int k) {
  using P = PkOut<LMAX>;
  const int m = k >> 1;
  const int odd_at = P::EB + (m & 15) * P::STR1 + (m >> 4);
  return o[(k & 1) ? odd_at : m];  // select, one load (no divergent branch)
}

template <int M, bool BLUE, int LMAX>
__device__ __forceinline__ void pk_split2(const double2* buf, const BlueTables& bt, double* oa, double* ob, int t,
                                          int T, const double2* pfa_u0 = nullptr) {
  using P = PkOut<LMAX>;
  const int N = bt.N;
  const double hs = 0.5 * bt.scale;
  for (int l = t; 2 * l <= N - 1; l += T) {
    const int m = l == 0 ? 0 : N - l;
    double2 zl, zm;
    if constexpr (pfa_len(M)) {
      zl = pfa_get<M>(buf, bt, l, pfa_u0);
      zm = pfa_get<M>(buf, bt, m, pfa_u0);
    } else {
      zl = pre<BLUE>(buf[pad<M>(l)], bt, l);
      zm = pre<BLUE>(buf[pad<M>(m)], bt, m);
    }
    if (l >= 1) {
      oa[l] = hs * (zm.y - zl.y);
      ob[l] = hs * (zl.x - zm.x);
    }
    if (2 * l + 1 <= N - 1) {
      const double f = l == 0 ? 0.25 : 0.5;
      const int q = P::EB + (l & 15) * P::STR1 + (l >> 4);
      oa[q] = f * (zl.x + zm.x);
      ob[q] = f * (zl.y + zm.y);
    }
  }
}

// Odd-output scans of `nlines` output lines (stride LS), one warp per line.
template <int LMAX>
__device__ __forceinline__ void odd_scans2(double* o, int LS, int nlines, const BlueTables& bt) {
  using P = PkOut<LMAX>;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  const int cnt = bt.N / 2;
  const double sc = bt.scale;
  for (int s = w; s < nlines; s += nw) {
    double* q = o + (size_t)s * LS + P::EB + lane;
    double v[16];
    double acc = 0.0;
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      v[i] = (16 * lane + i < cnt) ? q[i * P::STR1] : 0.0;
      acc += v[i];
      v[i] = acc;
    }
    double inc = acc;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, inc, d);
      if (lane >= d) inc += y;
    }
    const double off = inc - acc;
#pragma unroll
    for (int i = 0; i < 16; ++i)
      if (16 * lane + i < cnt) q[i * P::STR1] = (v[i] + off) * sc;
  }
}

// cp.async copy of `nl` contiguous lines of n doubles (src) into smem lines of
// stride LS (dst); 16-byte copies when n and both bases allow it.
__device__ __forceinline__ void stage_lines(double* dst, int LS, const double* src, int nl, int n) {
  const int nt = blockDim.x;
  const bool v16 = ((n | LS) & 1) == 0 && (((unsigned long long)src | (unsigned long long)__cvta_generic_to_shared(dst)) & 15) == 0;
  for (int h = 0; h < nl; ++h) {
    double* d = dst + (size_t)h * LS;
    const double* q = src + (size_t)h * n;
    if (v16) {
      for (int j = 2 * threadIdx.x; j < n; j += 2 * nt) cp_async16(d + j, q + j);
    } else {
      for (int j = threadIdx.x; j < n; j += nt) cp_async8(d + j, q + j);
    }
  }
}

// ---------------------------------------------------------------------------
// TMA bulk staging (cp.async.bulk + mbarrier transaction counts): ONE thread
// issues a whole contiguous line per instruction instead of every thread
// issuing 16-byte cp.async copies.  Usage: bulk_init(mb) by the CTA at start
// (thread 0), stage_lines_bulk(...) right after, and stage_lines_wait(...) by
// every thread once the CTA has passed a barrier after the init.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void bulk_init(unsigned long long* mb, int n, bool lead = threadIdx.x == 0) {
  if (lead) {
    for (int i = 0; i < n; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(mb + i)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
}

__device__ __forceinline__ void mbar_wait(unsigned long long* mb, unsigned parity) {
  asm volatile(
      "{\n"
      ".reg .pred P1;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(mb)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void mbar_expect(unsigned long long* mb, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(mb)), "r"(bytes) : "memory");
}

// one contiguous global -> smem copy (16-byte aligned, bytes % 16 == 0)
__device__ __forceinline__ void bulk_copy(void* dst, const void* src, unsigned bytes, unsigned long long* mb) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(mb))
               : "memory");
}

// Stage nl contiguous lines of n doubles into smem lines of stride LS: bulk
// copies completing on mb when n, LS and both bases are 16-byte friendly
// (returns true, CTA-uniform), else per-thread cp.async (caller commits).
__device__ __forceinline__ bool stage_lines_bulk(double* dst, int LS, const double* src, int nl, int n,
                                                 unsigned long long* mb) {
  const bool v16 = ((n | LS) & 1) == 0 && (((unsigned long long)src | (unsigned long long)smem_u32(dst)) & 15) == 0;
  if (!v16) {
    stage_lines(dst, LS, src, nl, n);
    return false;
  }
  if (threadIdx.x == 0 && nl > 0) {
    const unsigned bytes = (unsigned)n * 8u;
    mbar_expect(mb, bytes * nl);
    for (int h = 0; h < nl; ++h) bulk_copy(dst + (size_t)h * LS, src + (size_t)h * n, bytes, mb);
  }
  return true;
}

// Every thread: the lines of stage_lines_bulk have landed and are visible
// (bulk: the mbarrier phase; fallback: this thread's cp.async + a CTA barrier).
__device__ __forceinline__ void stage_lines_wait(bool bulk, unsigned long long* mb, int nl) {
  if (bulk) {
    if (nl > 0) mbar_wait(mb, 0);
  } else {
    cp_async_wait_all();
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Direct row pass of a rank-1 mask (separable fused pipeline): the four rows
// src[h] (smem, stride LS, length n2) are AR-extended horizontally
// (boundary.hpp:56-62) into ext (stride LSX >= n2 + 2 q2 + 9, LSX = 4 mod
// 16), then correlated with the row taps w (2 Q + 1), blur.hpp:39-52 along one
// axis: outT[c * n1 + h] = sum_u w_u ext[h][c + u], c < n2, h < nl — stored
// transposed (the column pass reads a column contiguously), 4 lanes = one
// 32-byte sector.  Lane (cb, h) computes the 9 consecutive outputs of row h
// starting at 9 cb (9 cb + 4 h hits 16 distinct 8-byte slots per half warp).
// resident CTAs per SM the separable row/column kernels are compiled for
#ifndef DBX_SEP_MINB
#define DBX_SEP_MINB 2
#endif

__host__ __device__ constexpr int sep_lsx(int n2, int q2) {
  const int e = n2 + 2 * q2 + 9;
  return e + ((4 - e % 16) + 16) % 16;
}

__device__ __forceinline__ void sep_extend_rows(const double* src, int LS, double* ext, int LSX, int n2, int q2,
                                                int nl) {
  // interior copies (no per-element division or boundary test), then the
  // 2 q2 mirrored samples per row
  for (int h = 0; h < 4; ++h) {
    const double* x = src + h * LS;
    double* e = ext + h * LSX + q2;
    if (h < nl) {
      for (int j = threadIdx.x; j < n2; j += blockDim.x) e[j] = x[j];
    } else {
      for (int j = threadIdx.x; j < n2; j += blockDim.x) e[j] = 0.0;
    }
  }
  for (int idx = threadIdx.x; idx < 8 * q2; idx += blockDim.x) {
    const int h = idx / (2 * q2), m = idx - h * 2 * q2;  // m < q2: left sample q2 - m; else right
    const double* x = src + h * LS;
    double v = 0.0;
    int jp;
    if (m < q2) {
      const int k = q2 - m;  // f_{-k} = 2 f_0 - f_k
      jp = q2 - k;
      if (h < nl) v = 2.0 * x[0] - x[k];
    } else {
      const int k = m - q2 + 1;  // f_{n-1+k} = 2 f_{n-1} - f_{n-1-k}
      jp = q2 + n2 - 1 + k;
      if (h < nl) v = 2.0 * x[n2 - 1] - x[n2 - 1 - k];
    }
    ext[h * LSX + jp] = v;
  }
}

template <int Q>
__device__ __forceinline__ void sep_row_stencil_T(const double* ext, int LSX, const ConvTables& ct, int n2,
                                                  int nl, double* outT, int n1) {
  constexpr int R = 9, NTAP = 2 * Q + 1;
  const int h = threadIdx.x & 3;
  const int nblk = (n2 + R - 1) / R;
  for (int cb = threadIdx.x >> 2; cb < nblk; cb += blockDim.x >> 2) {
    const int c0 = cb * R;
    const double* src = ext + h * LSX + c0;
    double acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = 0.0;
#pragma unroll
    for (int s = 0; s < R + 2 * Q; ++s) {
      const double z = src[s];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = s - r;
        if (t >= 0 && t < NTAP) acc[r] = fma(ct.sepr_v[t], z, acc[r]);
      }
    }
    if (h < nl) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (c0 + r < n2) outT[(size_t)(c0 + r) * n1 + h] = acc[r];
    }
  }
}

// Q dispatch of the compiled separable row-tap counts (conv_sep_supported).
__device__ __forceinline__ void sep_row_pass(const double* ext, int LSX, const ConvTables& ct, int q2, int n2, int nl,
                                             double* outT, int n1) {
  if (q2 == 15) sep_row_stencil_T<15>(ext, LSX, ct, n2, nl, outT, n1);
  else if (q2 == 7) sep_row_stencil_T<7>(ext, LSX, ct, n2, nl, outT, n1);
}

template <typename K>
bool set_smem(K kernel, size_t bytes) {
  if (bytes > 227 * 1024) return false;
  if (bytes > 48 * 1024)
    return cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) == cudaSuccess;
  return true;
}


}  // namespace
}  // namespace dbx
