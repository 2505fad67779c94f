// dst.cu — separate-pass AR / SineI transforms (tensor_apply, precondition_apply,
// and the D-Landweber iteration when the fused row pipelines do not apply) in
// packed real form: TWO image lines per complex N-point DFT (sine pre-twiddle,
// conjugate-symmetric split, odd-output prefix scan — spectral_common.cuh).
//
// The N-point DFT (N = m+1 for the SineI kind, N = n-1 for the AR kinds) has
// three cores, chosen per axis on the host:
//   CORE_DIRECT  M = N, N smooth (prime factors <= 31): one mixed-radix FFT;
//   CORE_BLUE    M = 2^k >= 2N-1: Bluestein chirp-z (FFT, kernel multiply, IFFT);
//   CORE_RADER   M = N-1, N prime with N-1 smooth (8191 for C5): Rader's cyclic
//                convolution over the generator order (FFT, kernel, IFFT).
// The DST outputs overwrite the FFT line in place (two real lines of doubles),
// so a line costs padded_len(M) * 16 bytes of shared memory and nothing more:
// M = 8190 / 8192 lines (C5, 147 KB) fit one CTA.
//
// Replaces (reference): sine1_forward + r2r RODFT00 (transforms.hpp:114-121,
// 28-53), ar_forward / ar_inverse (transforms.hpp:148-173), tensor_map /
// tensor_apply (transforms.hpp:179-221), filter_apply AR branch
// (spectral.hpp:161-165).
#include <cuda_runtime.h>

#include <cstdlib>

#include "spectral_common.cuh"

namespace dbx {

namespace {

#ifdef DBX_DST_STOCKHAM
constexpr bool kDstCt = false;
#else
constexpr bool kDstCt = true;
#endif
#ifdef DBX_DST_CT_BLUE
constexpr bool kDstCtBlue = true;
#else
constexpr bool kDstCtBlue = false;
#endif

// One-line-per-CTA rows (Rader 8190 for C5, prime-factor 2047 for C4): the
// two input rows land in the line buffer by two TMA bulk copies, then the
// fill reads them from shared memory (pkc_fill_staged) instead of exposing
// the global-load latency of every unrolled group (-DDBX_DST_STAGE=0: A/B).
#ifndef DBX_DST_STAGE
#define DBX_DST_STAGE 1
#endif
constexpr bool kDstStage = DBX_DST_STAGE != 0;

// Threads of the one-line CTAs at M >= 8000 (C5's Rader 8190): 640 = 20
// warps puts the in-place CT levels (630 / 1170 / 546 / 2730 / 4095
// butterflies of radix 13 / 7 / 15 / 3 / 2) at 1 / 2 / 1 / 5 / 7 per thread
// instead of 2 / 3 / 2 / 6 / 8 at 512.
#ifndef DBX_DST_BIG_T
#define DBX_DST_BIG_T 512
#endif
constexpr int kDstBigT = DBX_DST_BIG_T;

template <int M, int CORE>
struct DstCfg {
  // PFA lines: one line per CTA, 256 threads (23 x 11 = 253 butterflies of
  // the widest column level)
  static constexpr int T = CORE == CORE_PFA ? 256 : M >= 8000 ? kDstBigT : line_threads(M, dst_per(M));
  static constexpr int G = CORE == CORE_PFA ? 1 : lines_for(M, kDstBudget, dst_per(M));  // FFT lines per CTA
  static constexpr int NT = T * G;
  // double2 per FFT line (PFA: one spare slot, so the two staged raw rows of
  // n = M + 1 doubles fit the line)
  static constexpr int LINE = CORE == CORE_PFA ? M + 1 : padded_len(M);
  // one-line CTAs stage their two input rows with TMA (pkc_fill_staged)
  static constexpr bool STAGE = G == 1 && (CORE == CORE_RADER || CORE == CORE_PFA) && kDstStage;
  static constexpr int LO = LINE;                                 // output line stride (doubles)
  // the Rader convolution core runs the in-place Cooley-Tukey ct_convolve
  // (C5 8190: transform class 146 -> 131 ms per run); Bluestein keeps the two
  // Stockham FFTs (C4 4096 = 8^4: 13.7 vs 15.4 ms with CT).  -DDBX_DST_STOCKHAM
  // forces Stockham, -DDBX_DST_CT_BLUE forces CT for Bluestein too (A/B).
  static constexpr bool CT = (CORE == CORE_RADER || (CORE == CORE_BLUE && kDstCtBlue)) && kDstCt;
  static constexpr int TWN = CORE == CORE_PFA ? fft::ct_twiddles_needed(Pfa<M>::R)
                             : CT ? fft::ct_twiddles_needed(M) : fft::twiddles_needed(M);
  static constexpr size_t base = (size_t)G * LINE * 16;
  static constexpr bool TW = base + (size_t)TWN * 16 <= kSmemCap;
  static constexpr size_t bytes = base + (TW ? (size_t)TWN * 16 : 0);
  static constexpr int NMAX = CORE == CORE_BLUE ? M / 2 + 1 : M + 1;  // N <= NMAX
  static constexpr int PS = ((NMAX - 1) / 2 + 1 + T - 1) / T;         // split items per thread
  // resident CTAs per SM the register budget is sized for, only when asked
  // (-DDBX_DST_MINB4096=3: the Bluestein 4096 lines of C4 at 80 registers —
  // 1.2 KB of spills, not kept).  An explicit minimum of 1 is NOT neutral: it
  // lets ptxas take 156 registers for dst_rows<4096> (one CTA per SM, C4
  // 21.8 -> 27.3 ms per run), so the default is the one-argument form.
#ifdef DBX_DST_MINB4096
  static constexpr int MINB = (M == 4096 && CORE == CORE_BLUE) ? DBX_DST_MINB4096 : 1;
#endif
};
#ifdef DBX_DST_MINB4096
#define DBX_DST_BOUNDS __launch_bounds__(DstCfg<M, CORE>::NT, DstCfg<M, CORE>::MINB)
#elif defined(DBX_PFA_MINB)
// PFA lines (32 KB each) at DBX_PFA_MINB CTAs per SM (A/B of the register cap)
#define DBX_DST_BOUNDS __launch_bounds__(DstCfg<M, CORE>::NT, CORE == CORE_PFA ? DBX_PFA_MINB : 0)
#else
#define DBX_DST_BOUNDS __launch_bounds__(DstCfg<M, CORE>::NT)
#endif

// buffer position of z_j and the DFT output Z_l for each core
template <int M, int CORE>
__device__ __forceinline__ double2 pkc_get(const double2* buf, const BlueTables& bt, int l, double2 A0,
                                           const double2* u0 = nullptr) {
  if constexpr (CORE == CORE_PFA) {
    return pfa_get<M>(buf, bt, l, u0);
  } else if constexpr (CORE == CORE_RADER) {
    if (l == 0) return A0;
    return buf[pad<M>(__ldg(bt.ridx + l))];
  } else if constexpr (CORE == CORE_BLUE) {
    return cmul(buf[pad<M>(l)], __ldg(bt.chirp + l));
  } else {
    return buf[pad<M>(l)];
  }
}

// Fill one FFT line with z_j = y^a_j + i y^b_j (pk_fill), placed per core;
// sd(h, j) = (x^h_j + x^h_{N-j}, x^h_j - x^h_{N-j}), j in [1, N/2].
template <int M, int CORE>
__device__ __forceinline__ void pkc_put(double2* buf, const BlueTables& bt, int j, double2 z) {
  if constexpr (CORE == CORE_RADER || CORE == CORE_PFA) {
    // Rader: a_p = z_{g^p}; PFA: the Good-Thomas input map into the row
    // layout (dlog is a bijection onto the line's slots)
    buf[pad<M>(__ldg(bt.dlog + j))] = z;
  } else if constexpr (CORE == CORE_BLUE) {
    buf[pad<M>(j)] = cmul(z, __ldg(bt.chirp + j));
  } else {
    buf[pad<M>(j)] = z;
  }
}
// positions no pair covers: 0, and the Bluestein zero padding [N, M)
template <int M, int T, int CORE>
__device__ __forceinline__ void pkc_zero_fill(double2* buf, const BlueTables& bt, int t) {
  if constexpr (CORE != CORE_RADER) {
    if (t == 0) buf[pad<M>(0)] = make_double2(0.0, 0.0);
    if constexpr (CORE == CORE_BLUE)
      for (int p = bt.N + t; p < M; p += T) buf[pad<M>(p)] = make_double2(0.0, 0.0);
  }
}

template <int M, int T, int CORE, typename F>
__device__ __forceinline__ void pkc_fill(double2* buf, const BlueTables& bt, int t, F sd) {
  const int N = bt.N, H = N / 2;
  auto put = [&](int j, double2 z) { pkc_put<M, CORE>(buf, bt, j, z); };
  pkc_zero_fill<M, T, CORE>(buf, bt, t);
  // U positions per thread in flight: every global load of a group is issued
  // before the first shared-memory store (the loads cannot move above the
  // stores on their own: generic pointers may alias)
  constexpr int U = 4;
  for (int j0 = 1 + t; j0 <= H; j0 += U * T) {
    double s[U];
    double2 A[U], B[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * T;
      if (j <= H) {
        s[u] = __ldg(bt.sn + j);
        A[u] = sd(0, j);
        B[u] = sd(1, j);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * T;
      if (j <= H) {
        put(j, make_double2(fma(s[u], A[u].x, 0.5 * A[u].y), fma(s[u], B[u].x, 0.5 * B[u].y)));
        if (N - j != j) put(N - j, make_double2(fma(s[u], A[u].x, -0.5 * A[u].y), fma(s[u], B[u].x, -0.5 * B[u].y)));
      }
    }
  }
}


// pkc_fill from the two raw rows staged in the line itself (xs[0, n) = row a,
// xs[n, 2n) = row b, TMA-landed on mb): the scatter indices and sine weights
// are fetched while the copies fly, every read of the rows lands in
// registers, one barrier, then the scatter over the same storage.  The
// arithmetic is pkc_fill's (sd(h, j) on the same values), so the line is
// bit-identical.
template <int M, int T, int CORE, typename F>
__device__ __forceinline__ void pkc_fill_staged(double2* buf, const BlueTables& bt, int t, unsigned long long* mb,
                                                F sd) {
  static_assert(CORE == CORE_RADER || CORE == CORE_PFA, "scatter cores only");
  const int N = bt.N, H = N / 2;
  constexpr int PF = ((M + 1) / 2 + T - 1) / T;
  int pj[PF], pm[PF];
  double s[PF];
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int j = 1 + t + i * T;
    if (j <= H) {
      pj[i] = __ldg(bt.dlog + j);
      pm[i] = __ldg(bt.dlog + N - j);
      s[i] = __ldg(bt.sn + j);
    }
  }
  __syncthreads();  // the mbarrier init (thread 0) is visible
  mbar_wait(mb, 0);
  double2 zj[PF], zm[PF];
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int j = 1 + t + i * T;
    if (j <= H) {
      const double2 A = sd(0, j), B = sd(1, j);
      zj[i] = make_double2(fma(s[i], A.x, 0.5 * A.y), fma(s[i], B.x, 0.5 * B.y));
      zm[i] = make_double2(fma(s[i], A.x, -0.5 * A.y), fma(s[i], B.x, -0.5 * B.y));
    }
  }
  __syncthreads();
  pkc_zero_fill<M, T, CORE>(buf, bt, t);
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int j = 1 + t + i * T;
    if (j <= H) {
      buf[pad<M>(pj[i])] = zj[i];
      if (N - j != j) buf[pad<M>(pm[i])] = zm[i];
    }
  }
}

// Refill the FFT line from values that live in the line itself (the outputs
// of a previous transform, val(h, k) = value k of new line h): every read
// lands in registers (PF pairs per thread), then a barrier, then the scatter.
template <int M, int T, int CORE, int PF, typename V>
__device__ __forceinline__ void pkc_refill(double2* buf, const BlueTables& bt, int t, V val) {
  const int N = bt.N, H = N / 2;
  double2 zj[PF], zm[PF];
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int j = 1 + t + i * T;
    if (j <= H) {
      const double s = __ldg(bt.sn + j);
      const double aj = val(0, j), am = val(0, N - j), bj = val(1, j), bm = val(1, N - j);
      const double2 A = make_double2(aj + am, aj - am), B = make_double2(bj + bm, bj - bm);
      zj[i] = make_double2(fma(s, A.x, 0.5 * A.y), fma(s, B.x, 0.5 * B.y));
      zm[i] = make_double2(fma(s, A.x, -0.5 * A.y), fma(s, B.x, -0.5 * B.y));
    }
  }
  __syncthreads();
  pkc_zero_fill<M, T, CORE>(buf, bt, t);
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int j = 1 + t + i * T;
    if (j <= H) {
      pkc_put<M, CORE>(buf, bt, j, zj[i]);
      if (N - j != j) pkc_put<M, CORE>(buf, bt, N - j, zm[i]);
    }
  }
}

// The N-point DFT of the G lines (every thread of the CTA calls it).
template <int M, int T, int G, int CORE>
__device__ __forceinline__ void pkc_core(double2* sm, double2* buf, const BlueTables& bt, const double2* tw, int t,
                                         double2* A0s, int g, double2* pfa_sm = nullptr) {
  cp_async_wait_all();
  __syncthreads();
  if constexpr (CORE == CORE_PFA) {
    static_assert(G == 1, "one PFA line per CTA");
    pfa_core<M, T>(buf, bt, tw, t, 0, pfa_sm);
  } else if constexpr (CORE == CORE_DIRECT && (M & 1)) {
    fft::fft_cta<M, -1, T, G>(sm, tw, threadIdx.x);
  } else if constexpr (DstCfg<M, CORE>::CT) {
    const int bar = G > 1 ? 1 + g : 0;
    fft::ct_convolve<M, T, fft::ct_kt(M)>(buf, tw, fft::ct_kt(M) ? bt.bctT : bt.bct, t, bar,
                                          CORE == CORE_RADER ? &A0s[g] : nullptr);
  } else {
    const int bar = G > 1 ? 1 + g : 0;
    fft::fft<M, -1, T>(buf, tw, t, bar);
    if constexpr (CORE != CORE_DIRECT) {
      if constexpr (CORE == CORE_RADER) {
        if (t == 0) A0s[g] = buf[pad<M>(0)];  // X_0 = sum of a (z_0 = 0)
      }
      constexpr int U = 4;  // kernel-spectrum loads in flight per thread
      for (int p0 = t; p0 < M; p0 += U * T) {
        double2 h[U];
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (p0 + u * T < M) h[u] = __ldg(bt.bhat + p0 + u * T);
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (p0 + u * T < M) buf[pad<M>(p0 + u * T)] = cmul(buf[pad<M>(p0 + u * T)], h[u]);
      }
      fft::line_sync(bar, T);
      fft::fft<M, +1, T>(buf, tw, t, bar);
    }
  }
}

// pk_split in place: the DST outputs of lines a, b overwrite the FFT line as
// doubles oa = [0, LO), ob = [LO, 2 LO).  Reads land in registers, then a
// CTA barrier, then the writes.
template <int M, int T, int CORE, int PS, int LO>
__device__ __forceinline__ void pkc_split(double2* buf, const BlueTables& bt, int t, double2 A0,
                                          const double2* u0 = nullptr) {
  const int N = bt.N;
  const double hs = 0.5 * bt.scale;
  double r[PS][4];
#pragma unroll
  for (int i = 0; i < PS; ++i) {
    const int l = t + i * T;
    if (2 * l <= N - 1) {
      const double2 zl = pkc_get<M, CORE>(buf, bt, l, A0, u0);
      const double2 zm = pkc_get<M, CORE>(buf, bt, l == 0 ? 0 : N - l, A0, u0);
      const double f = l == 0 ? 0.25 : 0.5;
      r[i][0] = hs * (zm.y - zl.y);   // X^a_{2l}
      r[i][1] = hs * (zl.x - zm.x);   // X^b_{2l}
      r[i][2] = f * (zl.x + zm.x);    // scan term of X^a_{2l+1}
      r[i][3] = f * (zl.y + zm.y);    // scan term of X^b_{2l+1}
    }
  }
  __syncthreads();
  double* oa = reinterpret_cast<double*>(buf);
  double* ob = oa + LO;
#pragma unroll
  for (int i = 0; i < PS; ++i) {
    const int l = t + i * T;
    if (2 * l <= N - 1) {
      if (l >= 1) {
        oa[2 * l] = r[i][0];
        ob[2 * l] = r[i][1];
      }
      if (2 * l + 1 <= N - 1) {
        oa[2 * l + 1] = r[i][2];
        ob[2 * l + 1] = r[i][3];
      }
    }
  }
}

// Odd-output scans of the CTA's 2G output lines (every thread calls it).
// With at least two warps per output line (the one-line CTAs of the long
// lengths: 16 warps, 2 lines) each line's scan is split into contiguous
// warp chunks (odd_scan_range) plus a prefix of the chunk totals, instead of
// one warp per line while the others wait at the barrier.
template <int G, int LINE, int LO>
__device__ __forceinline__ void pkc_scans(double2* sm, const BlueTables& bt) {
  __syncthreads();
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  constexpr int NLN = 2 * G;
  if (nw >= 2 * NLN) {
    __shared__ double tot[32];
    const int wpl = nw / NLN < 32 / NLN ? nw / NLN : 32 / NLN;  // warps per line
    const int s = w / wpl, wi = w - s * wpl, cnt = bt.N / 2;
    const int chunk = ((cnt + wpl - 1) / wpl + 31) / 32 * 32;
    const int lo = wi * chunk, hi = lo + chunk < cnt ? lo + chunk : cnt;
    double* o = reinterpret_cast<double*>(sm + (s >> 1) * LINE) + (s & 1) * LO;
    if (s < NLN) {
      const double tt = odd_scan_range(o, lo, hi, lane);
      if (lane == 0) tot[w] = tt;
    }
    __syncthreads();
    if (s < NLN) {
      double pre = 0.0;
      for (int i = 0; i < wi; ++i) pre += tot[s * wpl + i];
      const double sc = bt.scale;
      for (int m = lo + lane; m < hi; m += 32) o[2 * m + 1] = (o[2 * m + 1] + pre) * sc;
    }
  } else {
    for (int s = w; s < NLN; s += nw)
      odd_scan(reinterpret_cast<double*>(sm + (s >> 1) * LINE) + (s & 1) * LO, bt.N / 2, bt.scale, lane);
  }
  __syncthreads();
}

// (sum, difference) of the interior inputs at j and N-j for a transform kind
// (xj, xm: the raw line values there; ARINV subtracts the ramp terms,
// transforms.hpp:163-173, with p_j = 1 - j/(n-1)).
__device__ __forceinline__ double2 kind_sd(int kind, double xj, double xm, double x0, double xe, int j, double ri) {
  if (kind == DBX_KIND_ARINV)
    return make_double2(xj + xm - (x0 + xe), (xj - xm) - (x0 - xe) * fma(-2.0 * ri, (double)j, 1.0));
  return make_double2(xj + xm, xj - xm);
}

// Output k (0-based, line length n) of a transform kind from the DST outputs o.
__device__ __forceinline__ double kind_out(int kind, const double* o, int k, int n, double x0, double xe,
                                           double al, double ri) {
  if (kind == DBX_KIND_SINEI) return o[k + 1];
  if (kind == DBX_KIND_ARINV) return k == 0 ? al * x0 : (k == n - 1 ? al * xe : o[k]);
  const double a0 = x0 / al, a1 = xe / al;
  if (k == 0) return a0;
  if (k == n - 1) return a1;
  const double t1 = (double)k * ri;
  return o[k] + a0 * (1.0 - t1) + a1 * t1;
}

// ---------------------------------------------------------------------------
// Row pass: 2G rows per CTA (line g carries rows 2g, 2g+1), fused epilogue
// (store / Hadamard / r = g - v with ||r||^2 / x += tau v with norms).
template <int M, int CORE>
__global__ void DBX_DST_BOUNDS dst_rows(SpecArgs a) {
  DBX_PDL_WAIT();
  using C = DstCfg<M, CORE>;
  constexpr int T = C::T, G = C::G, NT = C::NT;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double red[32];
  __shared__ double2 A0s[G];
  __shared__ double ends[G][4];
  __shared__ double2 pfa_sm[2 * (CORE == CORE_PFA ? Pfa<M>::N1 : 1)];  // PFA: column u0 and Rader sums
  const int g = threadIdx.x / T, t = threadIdx.x - g * T;
  double2* buf = sm + g * C::LINE;
  const BlueTables& bt = a.blue2;
  const double2* tw = stage_twiddles<M, C::TW, C::TWN>(sm + G * C::LINE, bt.tw);
  const int n1 = a.n1, n = a.n2;
  int kind = a.kind1;
  const size_t N = (size_t)n1 * n;
  const int ra = blockIdx.x * 2 * G + 2 * g;
  const double* in = resolve_ptr(a.in, a.st, a.insel, b, a.batch, N);
  // L2 prefetch of the rows the CTA one resident wave ahead will read (the
  // one-line-per-CTA lengths: the fill's DRAM latency is not hidden by any
  // other resident CTA)
  if (a.pf > 0 && threadIdx.x == 0) {
    const size_t r0 = (size_t)(blockIdx.x + a.pf) * 2 * G;
    if (r0 < (size_t)n1) {
      const size_t nr = r0 + 2 * G <= (size_t)n1 ? 2 * G : n1 - r0;
      const unsigned bytes = (unsigned)(nr * n * sizeof(double)) & ~15u;
      asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(in + r0 * n), "r"(bytes) : "memory");
    }
  }
  const double* xa = ra < n1 ? in + (size_t)ra * n : nullptr;
  const double* xb = ra + 1 < n1 ? in + (size_t)(ra + 1) * n : nullptr;
  const bool sine = kind == DBX_KIND_SINEI;
  const double ri = bt.rinv;
  const int NL = bt.N;
  double a0, ae, b0, be;
  // TMA-staged fill (CTA-uniform condition): both rows present, AR kinds,
  // 16-byte rows that fit the line
  bool staged = false;
  if constexpr (C::STAGE) {
    __shared__ alignas(8) unsigned long long mb_fill;
    staged = xb && !sine && (n & 1) == 0 && 2 * n <= 2 * C::LINE && ((reinterpret_cast<size_t>(xa) & 15) == 0);
    if (staged) {
      double* xs = reinterpret_cast<double*>(buf);
      if (threadIdx.x == 0) {
        bulk_init(&mb_fill, 1);
        mbar_expect(&mb_fill, (unsigned)n * 16u);
        bulk_copy(xs, xa, (unsigned)n * 8u, &mb_fill);
        bulk_copy(xs + n, xb, (unsigned)n * 8u, &mb_fill);
      }
      a0 = __ldg(xa); ae = __ldg(xa + n - 1); b0 = __ldg(xb); be = __ldg(xb + n - 1);
      pkc_fill_staged<M, T, CORE>(buf, bt, t, &mb_fill, [&](int hh, int j) {
        const double* x = xs + hh * n;
        return kind_sd(kind, x[j], x[NL - j], hh ? b0 : a0, hh ? be : ae, j, ri);
      });
    }
  }
  if (!staged) {
    a0 = (xa && !sine) ? xa[0] : 0.0; ae = (xa && !sine) ? xa[n - 1] : 0.0;
    b0 = (xb && !sine) ? xb[0] : 0.0; be = (xb && !sine) ? xb[n - 1] : 0.0;
    pkc_fill<M, T, CORE>(buf, bt, t, [&](int hh, int j) {
      const double* x = hh ? xb : xa;
      if (!x) return make_double2(0.0, 0.0);
      if (sine) return kind_sd(kind, x[j - 1], x[NL - j - 1], 0.0, 0.0, j, ri);
      return kind_sd(kind, x[j], x[NL - j], hh ? b0 : a0, hh ? be : ae, j, ri);
    });
  }
  pkc_core<M, T, G, CORE>(sm, buf, bt, tw, t, A0s, g, pfa_sm);
  pkc_split<M, T, CORE, C::PS, C::LO>(buf, bt, t, CORE == CORE_RADER ? A0s[g] : make_double2(0.0, 0.0), pfa_sm);
  pkc_scans<G, C::LINE, C::LO>(sm, bt);
  const double* o = reinterpret_cast<const double*>(buf);
  const double al = bt.alpha;
  if (a.kind2 >= 0) {
    // kind1, x d (the CTA's rows of the filter grid), kind2 on the same rows:
    // the column half of D = T diag(d) T~ on transposed images in one pass
    // (AR kinds only; the intermediate never leaves shared memory)
    const double* dd = a.d + (size_t)b * a.dstride;
    const double* da = xa ? dd + (size_t)ra * n : nullptr;
    const double* db = xb ? dd + (size_t)(ra + 1) * n : nullptr;
    auto val = [&](int hh, int k) {
      const double* dr = hh ? db : da;
      if (!dr) return 0.0;
      return kind_out(kind, o + hh * C::LO, k, n, hh ? b0 : a0, hh ? be : ae, al, ri) * __ldg(dr + k);
    };
    if (t < 4) ends[g][t] = val(t >> 1, (t & 1) ? n - 1 : 0);
    constexpr int PF = (C::NMAX / 2 + T - 1) / T;
    pkc_refill<M, T, CORE, PF>(buf, bt, t, val);
    a0 = ends[g][0]; ae = ends[g][1]; b0 = ends[g][2]; be = ends[g][3];
    kind = a.kind2;
    pkc_core<M, T, G, CORE>(sm, buf, bt, tw, t, A0s, g, pfa_sm);
    pkc_split<M, T, CORE, C::PS, C::LO>(buf, bt, t, CORE == CORE_RADER ? A0s[g] : make_double2(0.0, 0.0), pfa_sm);
    pkc_scans<G, C::LINE, C::LO>(sm, bt);
  }
  if (a.tout && a.epi == SPEC_STORE) {
    // transposed store (replaces a transpose launch between the row passes
    // of D): the line's two rows leave as one 16-byte pair per column; the
    // CTAs of adjacent row pairs run in the same wave, so L2 completes the
    // sectors before they are written back
    double* y = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N));
    const double x0a = a0, xea = ae, x0b = b0, xeb = be;
    if (ra + 1 < n1 && (n1 & 1) == 0) {
      for (int k = t; k < n; k += T)
        *reinterpret_cast<double2*>(y + (size_t)k * n1 + ra) =
            make_double2(kind_out(kind, o, k, n, x0a, xea, al, ri), kind_out(kind, o + C::LO, k, n, x0b, xeb, al, ri));
    } else if (ra < n1) {
      for (int k = t; k < n; k += T) {
        y[(size_t)k * n1 + ra] = kind_out(kind, o, k, n, x0a, xea, al, ri);
        if (ra + 1 < n1) y[(size_t)k * n1 + ra + 1] = kind_out(kind, o + C::LO, k, n, x0b, xeb, al, ri);
      }
    }
    return;
  }
  Epi e = make_epi(a, b, N);
  if (a.kind2 >= 0) e.d = nullptr;
  for (int hh = 0; hh < 2; ++hh) {
    const int r = ra + hh;
    if (r >= n1) continue;
    const double* oh = o + hh * C::LO;
    const double x0 = hh ? b0 : a0, xe = hh ? be : ae;
    epi_row<4>(e, (size_t)r * n, n, t, T, [&](int k) { return kind_out(kind, oh, k, n, x0, xe, al, ri); });
  }
  write_partials<NT>(a, e, red, b);
}

// ---------------------------------------------------------------------------
// Column pass: 2G adjacent columns per CTA (line g carries columns 2g, 2g+1;
// row segments of 2G doubles).  kind1, then (kind2 >= 0) the middle Hadamard
// by the d column and kind2 — the whole column half of D = T diag(d) T~ — with
// the middle product parked in the output array (the CTA's own columns).
// ---------------------------------------------------------------------------
// Column pass: 2G adjacent columns per CTA (line g carries columns 2g, 2g+1;
// row segments of 2G doubles), transform a.kind1 with the STORE / Hadamard
// epilogue.  The column half of D = T diag(d) T~ is two launches (the host
// side, launch_dst_cols): T~ with the Hadamard by d into the output array, then
// T in place on it.
template <int M, int CORE>
__global__ void DBX_DST_BOUNDS dst_cols(SpecArgs a) {
  DBX_PDL_WAIT();
  using C = DstCfg<M, CORE>;
  constexpr int T = C::T, G = C::G, NT = C::NT;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double2 A0s[G];
  __shared__ double e0[2 * G], e1[2 * G];
  __shared__ double2 pfa_sm[2 * (CORE == CORE_PFA ? Pfa<M>::N1 : 1)];  // PFA: column u0 and Rader sums
  const int g = threadIdx.x / T, t = threadIdx.x - g * T;
  double2* buf = sm + g * C::LINE;
  const BlueTables& bt = a.blue1;
  const double2* tw = stage_twiddles<M, C::TW, C::TWN>(sm + G * C::LINE, bt.tw);
  const int n = a.n1, n2 = a.n2;
  const size_t N = (size_t)n * n2;
  const int c0 = blockIdx.x * 2 * G;
  const int ncol = n2 - c0 < 2 * G ? n2 - c0 : 2 * G;
  double* out = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N));
  const double* in = resolve_ptr(a.in, a.st, a.insel, b, a.batch, N);
  const double ri = bt.rinv, al = bt.alpha;
  const int kind = a.kind1;
  const bool sine = kind == DBX_KIND_SINEI;
  if (threadIdx.x < 2 * G) {
    const int s = threadIdx.x, c = c0 + s;
    e0[s] = (s < ncol && !sine) ? in[c] : 0.0;
    e1[s] = (s < ncol && !sine) ? in[(size_t)(n - 1) * n2 + c] : 0.0;
  }
  __syncthreads();
  const int ca = c0 + 2 * g;
  const double xa0 = e0[2 * g], xae = e1[2 * g], xb0 = e0[2 * g + 1], xbe = e1[2 * g + 1];
  const bool la = 2 * g < ncol, lb = 2 * g + 1 < ncol;
  const int NL = bt.N;
  pkc_fill<M, T, CORE>(buf, bt, t, [&](int hh, int j) {
    if (!(hh ? lb : la)) return make_double2(0.0, 0.0);
    const double* x = in + ca + hh;
    if (sine) return kind_sd(kind, x[(size_t)(j - 1) * n2], x[(size_t)(NL - j - 1) * n2], 0.0, 0.0, j, ri);
    return kind_sd(kind, x[(size_t)j * n2], x[(size_t)(NL - j) * n2], hh ? xb0 : xa0, hh ? xbe : xae, j, ri);
  });
  pkc_core<M, T, G, CORE>(sm, buf, bt, tw, t, A0s, g, pfa_sm);
  pkc_split<M, T, CORE, C::PS, C::LO>(buf, bt, t, CORE == CORE_RADER ? A0s[g] : make_double2(0.0, 0.0), pfa_sm);
  pkc_scans<G, C::LINE, C::LO>(sm, bt);
  // outputs: 2G adjacent columns per row (index s fastest)
  const bool had = a.epi == SPEC_HADAMARD && a.d;
  for (int idx = threadIdx.x; idx < n * 2 * G; idx += NT) {
    const int k = idx / (2 * G), s = idx - k * (2 * G);
    if (s >= ncol) continue;
    const double* o = reinterpret_cast<const double*>(sm + (s >> 1) * C::LINE) + (s & 1) * C::LO;
    double v = kind_out(kind, o, k, n, e0[s], e1[s], al, ri);
    const size_t at = (size_t)k * n2 + c0 + s;
    if (had) v *= a.d[(size_t)b * a.dstride + at];
    out[at] = v;
  }
}

// L2 prefetch of the next resident wave's rows in the one-line-per-CTA row
// passes (C5: 125.8 -> 124.6 ms transform class per run); DBX_DST_PF=0 disables
static bool dst_pf_enabled() {
  static const bool on = [] { const char* e = getenv("DBX_DST_PF"); return !(e && e[0] == '0'); }();
  return on;
}

template <int L, int CORE>
int rows_launch(const SpecArgs& a, cudaStream_t s) {
  using C = DstCfg<L, CORE>;
  static AttrOnce attr;
  if (!attr.ensure(dst_rows<L, CORE>, C::bytes)) return -1;
  dim3 grid((a.n1 + 2 * C::G - 1) / (2 * C::G), a.batch);
  SpecArgs b = a;
  b.pf = 0;
  if (C::G == 1 && dst_pf_enabled()) {
    static const int resident = [] {
      int dev = 0, sms = 0, occ = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, dst_rows<L, CORE>, C::NT, C::bytes);
      return sms * (occ > 0 ? occ : 1);
    }();
    b.pf = resident;
  }
  launch_k(dst_rows<L, CORE>, grid, C::NT, C::bytes, s, b);
  return (int)grid.x;
}

template <int L, int CORE>
int cols_launch(const SpecArgs& a, cudaStream_t s) {
  using C = DstCfg<L, CORE>;
  static AttrOnce attr;
  if (!attr.ensure(dst_cols<L, CORE>, C::bytes)) return -1;
  dim3 grid((a.n2 + 2 * C::G - 1) / (2 * C::G), a.batch);
  launch_k(dst_cols<L, CORE>, grid, C::NT, C::bytes, s, a);
  return (int)grid.x;
}

}  // namespace

#define DBX_DIRECT_LIST(X) X(15) X(31) X(63) X(255) X(1023) X(4095)
#define DBX_BLUE_LIST(X) X(16) X(32) X(64) X(128) X(256) X(512) X(1024) X(2048) X(4096) X(8192)
#define DBX_RADER_LIST(X) X(22) X(126) X(8190)
// prime-factor lengths N = N1 N2 (N1 <= 31 compiled radix, N2 prime, N2 - 1 a
// compiled CT length; pfa.cuh pfa_len): 2047 = 23 x 89 (C4), 511 = 7 x 73 (C2),
// 115 = 23 x 5 (tests: small lines)
#define DBX_PFA_LIST(X) X(2047) X(511) X(115)

int direct_supported_len(int N) {
#define X(L) if (N == (L)) return (L);
  DBX_DIRECT_LIST(X)
#undef X
  return 0;
}

int blue_supported_len(int need) {
  int best = 0;
#define X(L) if (best == 0 && (L) >= need) best = (L);
  DBX_BLUE_LIST(X)
#undef X
  return best;
}

int pfa_supported_len(int N) {
#define X(L) if (N == (L)) return (L);
  DBX_PFA_LIST(X)
#undef X
  return 0;
}

void pfa_factors(int N, int* N1, int* N2) {
  *N1 = 0;
  *N2 = 0;
#define X(L) if (N == (L)) { *N1 = Pfa<L>::N1; *N2 = Pfa<L>::N2; }
  DBX_PFA_LIST(X)
#undef X
}

int rader_supported_len(int M) {
#define X(L) if (M == (L)) return (L);
  DBX_RADER_LIST(X)
#undef X
  return 0;
}

static int dispatch(int core, int M, const SpecArgs& a, cudaStream_t s, bool rows) {
  if (core == CORE_DIRECT) {
#define X(L) if (M == (L)) return rows ? rows_launch<L, CORE_DIRECT>(a, s) : cols_launch<L, CORE_DIRECT>(a, s);
    DBX_DIRECT_LIST(X)
#undef X
  } else if (core == CORE_BLUE) {
#define X(L) if (M == (L)) return rows ? rows_launch<L, CORE_BLUE>(a, s) : cols_launch<L, CORE_BLUE>(a, s);
    DBX_BLUE_LIST(X)
#undef X
  } else if (core == CORE_PFA) {
#define X(L) if (M == (L)) return rows ? rows_launch<L, CORE_PFA>(a, s) : cols_launch<L, CORE_PFA>(a, s);
    DBX_PFA_LIST(X)
#undef X
  } else {
#define X(L) if (M == (L)) return rows ? rows_launch<L, CORE_RADER>(a, s) : cols_launch<L, CORE_RADER>(a, s);
    DBX_RADER_LIST(X)
#undef X
  }
  return -1;
}

int launch_dst_rows(const SpecArgs& a, cudaStream_t s) { return dispatch(a.blue2.core, a.blue2.M, a, s, true); }
// kind2 >= 0: kind1 with the Hadamard by d (when given) into out, then kind2
// in place on out.
int launch_dst_cols(const SpecArgs& a, cudaStream_t s) {
  if (a.kind2 < 0) return dispatch(a.blue1.core, a.blue1.M, a, s, false);
  SpecArgs p = a;
  p.kind2 = -1;
  p.epi = a.d ? SPEC_HADAMARD : SPEC_STORE;
  const int r = dispatch(a.blue1.core, a.blue1.M, p, s, false);
  if (r < 0) return r;
  p.kind1 = a.kind2;
  p.in = a.out;
  p.insel = a.outsel;
  p.epi = SPEC_STORE;
  return dispatch(a.blue1.core, a.blue1.M, p, s, false);
}

}  // namespace dbx
