// fused.cu — fused row pipelines of the preconditioned iteration (FFT-form
// blur + FFT-form AR transform).  A CTA owns four image rows (two packed
// real-FFT conv lines of length L2 and, where a transform follows, two packed
// real DST lines of length M, two rows per line); every stage stays
// in shared memory between the passes that used to be separate launches:
//
//   rows_ainv_tt      : Y (A' r spectrum) -> inverse row FFT -> s = A'r rows
//                       -> T~ (AR inverse transform, DST-I) along the rows -> u
//   rows_t_axpy_afwd  : v -> T along the rows -> x_k = x_{k-1} + tau*(.) with
//                       ||x||^2, ||x - f||^2 partials -> AR-extend x_k rows ->
//                       forward row FFT -> Z (spectrum for A x_k)
//   rows_ainv_resid   : Y (A x_k spectrum) -> inverse row FFT -> r = g - A x_k
//                       with ||r||^2 partials -> AR-extend r rows -> forward
//                       row FFT -> Z' (spectrum for A' r of the next iteration)
//
// Together with conv_col (twice) and dst_cols the iteration takes 6 launches
// + finalize instead of 9 + finalize, and x, r, s never make an extra HBM
// round trip.  Reference: the loop body of landweber_loop (solver.hpp:101-125)
// with apply (blur.hpp:75-83), precondition_apply (preconditioner.hpp:88-90).
#include <cuda_runtime.h>

#include <cstdlib>

#include "spectral_common.cuh"
#include "finalize.cuh"

namespace dbx {

namespace {

// Fused DST lines carry one radix-8 butterfly per thread also for the
// power-of-two Bluestein lengths (twice the threads of the separate-pass
// kernels): the fused shapes with Bluestein lines are single small images
// (C2: 512^2 -> 128 CTAs for 148 SMs), where per-CTA latency, not issue
// width, sets the kernel time.
__host__ __device__ constexpr int fused_dst_per(int) { return 8; }
// Threads per fused DST line (FUSED_TD_ODD overrides long odd lines, A/B).
#ifndef FUSED_TD_ODD
#define FUSED_TD_ODD 128  // A/B r1s2m: 96 (line_threads) 14972, 128 15455, 160 15152, 192 15209
#endif
__host__ __device__ constexpr int fused_td(int M) {
  // prime-factor lines (pfa.cuh, C2's 511 = 7 x 73): 128 threads (73 row
  // DFTs, 63 butterflies of the widest column level)
  return pfa_len(M) ? 128
         : (FUSED_TD_ODD > 0 && (M & 1) && M > 512) ? FUSED_TD_ODD : line_threads(M, fused_dst_per(M));
}

#ifndef DBX_TT_MINB
#define DBX_TT_MINB 3
#endif
#ifndef DBX_TC_MINB
#define DBX_TC_MINB 2
#endif
template <int L2, int M, bool BLUE>
struct Fused {
  static constexpr int TD = fused_td(M);   // threads per line
  static constexpr int NT = 2 * TD;                         // CTA = two FFT lines
  static constexpr int LC = padded_len(L2);                 // conv line (double2)
  static constexpr int LD = padded_len(M);                  // DST line (double2)
  static constexpr size_t kBudget = 115200;                 // two CTAs per SM (228 KB - reserved)
  static constexpr size_t TWD = (size_t)dst_twiddles_needed(M) * 16;     // staged twiddle prefixes
  static constexpr size_t TWC = (size_t)fft::twiddles_needed(L2) * 16;
  // ---- 4-row kernels (rows_ainv_tt, rows_t_axpy_afwd): two conv lines of
  // two packed rows each, then two packed DST lines of two rows each
  static constexpr int W4 = (LC > LD ? LC : LD) * 2;        // work region (double2)
  static constexpr int LMAX = BLUE ? M / 2 + 1 : M + 1;     // longest row n2
  static constexpr int LS = (LMAX + 1) / 2 * 2 + 4;         // smem row stride (doubles)
  static constexpr int LSO = ((LMAX > PkOut<LMAX>::OL ? LMAX : PkOut<LMAX>::OL) + 1) / 2 * 2 + 4;  // rows that receive DST outputs
  static constexpr size_t off_rows = (size_t)W4 * 16;       // 4 rows (stride LSO)
  static constexpr size_t off_x = off_rows + (size_t)4 * LSO * 8;  // 4 more rows (t_axpy)
  // rows_ainv_tt: twiddles after the rows
  static constexpr size_t tt_twd = off_x;
  static constexpr bool TT_TWD = tt_twd + TWD <= kBudget;
  static constexpr size_t tt_twc = tt_twd + (TT_TWD ? TWD : 0);
  static constexpr bool TT_TWC = tt_twc + TWC <= kBudget;
  static constexpr size_t tt_bytes = tt_twc + (TT_TWC ? TWC : 0);
  // separable rows_ainv_tt: no conv FFT, so no conv twiddles; DBX_TT_MINB = 3
  // also leaves the DST twiddles in global memory (L1) so three CTAs fit
  static constexpr bool TTS_TWD = DBX_TT_MINB < 3 && TT_TWD;
  static constexpr size_t tts_bytes = tt_twd + (TTS_TWD ? TWD : 0);
  // rows_t_axpy_afwd: v rows (then T output), x rows, twiddles if they fit
  // x rows of rows_t_axpy: stride LS, or (separable variant) LSXR with the
  // data at offset 16 and room for the in-place AR extension (q2 <= 15)
  static constexpr int LSXR = (16 + LMAX + 15 + 9) + ((4 - (16 + LMAX + 15 + 9) % 16) + 16) % 16;
  static constexpr int LSX_MAX = LSXR > LS ? LSXR : LS;
  static constexpr size_t ax_twd = off_x + (size_t)4 * LSX_MAX * 8;
  static constexpr bool AX_TWD = ax_twd + TWD <= kBudget;
  static constexpr size_t ax_twc = ax_twd + (AX_TWD ? TWD : 0);
  static constexpr bool AX_TWC = ax_twc + TWC <= kBudget;
  static constexpr size_t ax_bytes = ax_twc + (AX_TWC ? TWC : 0);
  static_assert((size_t)W4 * 16 >= (size_t)4 * LS * 8, "f rows are staged in the work region");
};

// Inverse packed real FFT of rows (ra, rb) from the half spectra Y -> buf
// (T threads on the line, thread index t).
template <int L2, int T>
__device__ __forceinline__ void conv_inv_load(double2* buf, const double2* __restrict__ Y, int ra, int rb,
                                              int n1, int Lh, int t) {
  constexpr int PF = (L2 / 2 + 1 + T - 1) / T;
  double2 A[PF], Bv[PF];
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int k = t + i * T;
    A[i] = make_double2(0.0, 0.0);
    Bv[i] = A[i];
    if (k < Lh) {
      if (ra < n1) A[i] = Y[(size_t)ra * y_stride(Lh) + k];
      if (rb < n1) Bv[i] = Y[(size_t)rb * y_stride(Lh) + k];
    }
  }
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int k = t + i * T;
    if (k < Lh) {
      buf[pad<L2>(k)] = make_double2(A[i].x - Bv[i].y, A[i].y + Bv[i].x);
      if (k > 0 && k < L2 - k) buf[pad<L2>(L2 - k)] = make_double2(A[i].x + Bv[i].y, Bv[i].x - A[i].y);
    }
  }
}

// Forward packed real FFT of two real rows held in shared memory (AR-extended
// horizontally on the fly, boundary.hpp:56-62) -> half spectra, stored
// transposed into Z ([k][row]) so the column pass reads each column
// contiguously.  Every thread of the CTA calls it (CTA-wide barriers).
template <int L2, int T>
__device__ __forceinline__ void conv_fwd_rows(double2* buf, const double* rowa, const double* rowb, int n2,
                                              int q2, const double2* tw, double2* Z, int ra, int rb, int n1,
                                              int Lh, int t, int bar) {
  const int wext = n2 + 2 * q2;
  const bool has_a = ra < n1, has_b = rb < n1;
  // the AR-extended rows are produced inside the first FFT stage's loads:
  // interior samples are plain copies; only the 2 q2 mirrored samples and the
  // zero tail take the (warp-local) boundary branch
  fft::fft_in<L2, -1, T>(buf, tw, t, bar, [&](int p) {
    const int j = p - q2;
    int jc = j < 0 ? -j : j >= n2 ? 2 * (n2 - 1) - j : j;
    jc = jc < 0 ? 0 : jc;
    double va = rowa[jc], vb = rowb[jc];
    if (j < 0 || j >= n2) {
      const int e = j < 0 ? 0 : n2 - 1;
      va = p < wext ? 2.0 * rowa[e] - va : 0.0;
      vb = p < wext ? 2.0 * rowb[e] - vb : 0.0;
    }
    return make_double2(has_a ? va : 0.0, has_b ? vb : 0.0);
  });
  const bool pair = has_b && ((ra | n1) & 1) == 0;  // rows ra, ra+1 adjacent and 32-byte aligned
  for (int k = t; k < Lh; k += T) {
    const double2 zk = buf[pad<L2>(k)], zm = buf[pad<L2>(k == 0 ? 0 : L2 - k)];
    const double2 za = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    const double2 zb = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
    if (pair) {
      st_pair(Z + (size_t)k * n1 + ra, za, zb);
    } else {
      if (has_a) Z[(size_t)k * n1 + ra] = za;
      if (has_b) Z[(size_t)k * n1 + rb] = zb;
    }
  }
}

// ---------------------------------------------------------------------------
// rows_ainv_tt: FOUR rows per CTA.  Conv line g (TD threads) inverts the
// spectra of rows 2g, 2g+1; DST line g then carries T~ of the same two rows
// (packed real DST).  u is written transposed (u^T[k][row], 32-byte sectors).
template <int L2, int M, bool BLUE, bool SEP = false>
__global__ void __launch_bounds__(Fused<L2, M, BLUE>::NT, SEP ? DBX_TT_MINB : 2) rows_ainv_tt(SpecArgs a) {
  DBX_PDL_WAIT();
  using F = Fused<L2, M, BLUE>;
  constexpr int NT = F::NT, TD = F::TD, LS = F::LSO, LMAX = F::LMAX;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double e0[4], e1[4];
  char* base = reinterpret_cast<char*>(sm);
  double* rowS = reinterpret_cast<double*>(base + F::off_rows);  // 4 rows: s, then T~ output
  const BlueTables& bt = a.blue2;
  const double2* twd =
      stage_twiddles<M, SEP ? F::TTS_TWD : F::TT_TWD>(reinterpret_cast<double2*>(base + F::tt_twd), bt.tw);
  const double2* twc =
      stage_twiddles<L2, F::TT_TWC && !SEP>(reinterpret_cast<double2*>(base + F::tt_twc), a.conv.tw2);
  const int n1 = a.n1, n2 = a.n2, Lh = a.conv.Lh;
  const size_t N = (size_t)n1 * n2;
  const int r0 = 4 * blockIdx.x;
  const int nl = n1 - r0 < 4 ? n1 - r0 : 4;
  const int g = threadIdx.x / TD, t = threadIdx.x - g * TD;
  PH_DECL
  if constexpr (SEP) {
    // separable pipeline: the column pass already produced s = A'r rows (real,
    // row-major in ybuf): stage them straight into the DST input rows
    __shared__ unsigned long long mbs[1];
    bulk_init(mbs, 1);
    const bool bs = stage_lines_bulk(rowS, LS, reinterpret_cast<const double*>(a.ybuf) + (size_t)b * N +
                                                   (size_t)r0 * n2, nl, n2, mbs);
    cp_async_commit();
    cp_async_wait_all();
    __syncthreads();
    stage_lines_wait(bs, mbs, nl);
    (void)twc;
    (void)Lh;
  } else {
    const int ra = r0 + 2 * g, rb = ra + 1;
    // A' r rows: inverse packed row FFT (conv line g = rows 2g, 2g+1)
    double2* cbuf = sm + g * F::LC;
    conv_inv_load<L2, TD>(cbuf, a.ybuf + (size_t)b * n1 * y_stride(Lh), ra, rb, n1, Lh, t);
    cp_async_wait_all();
    __syncthreads();
    PH(20)
    fft::fft<L2, +1, TD>(cbuf, twc, t, 1 + g);
    PH(21)
    for (int c = t; c < n2; c += TD) {
      const double2 v = cbuf[pad<L2>(c)];
      rowS[(2 * g) * LS + c] = v.x;
      rowS[(2 * g + 1) * LS + c] = v.y;
    }
    __syncthreads();
  }
  PH(22)
  if (threadIdx.x < 4) {
    e0[threadIdx.x] = rowS[threadIdx.x * LS];
    e1[threadIdx.x] = rowS[threadIdx.x * LS + n2 - 1];
  }
  // T~ along the rows (ar_inverse, transforms.hpp:163-173)
  const double ri = bt.rinv;
  double2* dbuf = sm + g * F::LD;
  // AR-inverse interior (s_j - s_0 p_j - s_{n-1} p_{n-1-j}; p_j = 1 - j/(n-1),
  // transforms.hpp:135-144, 163-173) as (sum, difference) of the pair j, N-j
  const int N2 = bt.N;
  const double xa0 = rowS[(2 * g) * LS], xae = rowS[(2 * g) * LS + n2 - 1];
  const double xb0 = rowS[(2 * g + 1) * LS], xbe = rowS[(2 * g + 1) * LS + n2 - 1];
  pk_fill<M, TD, BLUE>(dbuf, bt, t, [&](int hh, int j) {
    const int h = 2 * g + hh;
    if (h >= nl) return make_double2(0.0, 0.0);
    const double* L = rowS + h * LS;
    const double x0 = hh ? xb0 : xa0, xe = hh ? xbe : xae;
    const double lj = L[j], lm = L[N2 - j];
    return make_double2(lj + lm - (x0 + xe), (lj - lm) - (x0 - xe) * fma(-2.0 * ri, (double)j, 1.0));
  });
  PH(23)
  __shared__ double2 pfa_aux[2][2 * Pfa<M>::N1];  // prime-factor lines: u0 + Rader sums per line
  blue_core<M, TD, 2, BLUE>(sm, dbuf, bt, twd, t, pfa_aux[g]);
  PH(24)
  pk_split2<M, BLUE, LMAX>(dbuf, bt, rowS + (2 * g) * LS, rowS + (2 * g + 1) * LS, t, TD, pfa_aux[g]);
  __syncthreads();
  odd_scans2<LMAX>(rowS, LS, 4, bt);
  __syncthreads();
  PH(25)
  static_assert(NT % 4 == 0, "row-group mapping");
  const int h = threadIdx.x & 3;
  if (h < nl) {
    double* uT = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N)) + r0 + h;
    const double* o = rowS + h * LS;
    const double u0 = bt.alpha * e0[h], ue = bt.alpha * e1[h];
#pragma unroll 4
    for (int k = threadIdx.x >> 2; k < n2; k += NT / 4) {
      const double v = pk_at<LMAX>(o, k);  // o[0], o[n2-1] in bounds
      uT[(size_t)k * n1] = (k == 0) ? u0 : (k == n2 - 1) ? ue : v;
    }
  }
  PH(26)
}

// ---------------------------------------------------------------------------
// rows_t_axpy_afwd: FOUR rows per CTA.  T (packed DST) of the rows of v ->
// x_k = x_{k-1} + tau (.) with ||x||^2 / ||x - f||^2 partials -> forward
// packed row FFTs of x_k (conv line g = rows 2g, 2g+1) -> Z^T.
template <int L2, int M, bool BLUE, bool SEP = false>
__global__ void __launch_bounds__(Fused<L2, M, BLUE>::NT, 2) rows_t_axpy_afwd(SpecArgs a) {
  DBX_PDL_WAIT();
  using F = Fused<L2, M, BLUE>;
  constexpr int NT = F::NT, TD = F::TD, LS = F::LS, LSO = F::LSO, LMAX = F::LMAX;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double red[32];
  __shared__ double e0[4], e1[4];
  char* base = reinterpret_cast<char*>(sm);
  double* io = reinterpret_cast<double*>(base + F::off_rows);  // v rows, then T output
  double* stX = reinterpret_cast<double*>(base + F::off_x);    // x_{k-1} rows, then x_k
  const BlueTables& bt = a.blue2;
  const double2* twd = stage_twiddles<M, F::AX_TWD>(reinterpret_cast<double2*>(base + F::ax_twd), bt.tw);
  const double2* twc =
      stage_twiddles<L2, F::AX_TWC && !SEP>(reinterpret_cast<double2*>(base + F::ax_twc), a.conv.tw2);
  const int n1 = a.n1, n2 = a.n2, Lh = a.conv.Lh;
  const size_t N = (size_t)n1 * n2;
  const int r0 = 4 * blockIdx.x;
  const int nl = n1 - r0 < 4 ? n1 - r0 : 4;
  const int g = threadIdx.x / TD, t = threadIdx.x - g * TD;
  const double* xo = resolve_ptr(a.xold, a.st, a.xoldsel, b, a.batch, N) + (size_t)r0 * n2;
  const double* fimg = a.f ? a.f + (size_t)b * N + (size_t)r0 * n2 : nullptr;
  PH_DECL
  if (fimg && threadIdx.x < nl) prefetch_l2(fimg + (size_t)threadIdx.x * n2, (unsigned)n2 * 8);
  __shared__ unsigned long long mb[2];
  bulk_init(mb, 2);
  const bool bv = stage_lines_bulk(io, LSO, a.in + (size_t)b * N + (size_t)r0 * n2, nl, n2, mb);  // v rows
  cp_async_commit();
  constexpr int XS = SEP ? F::LSXR : LS, XO = SEP ? 16 : 0;  // x row stride / offset
  const bool bx = stage_lines_bulk(stX + XO, XS, xo, nl, n2, mb + 1);  // x_{k-1} rows
  cp_async_commit();
  cp_async_wait_group<1>();
  __syncthreads();
  stage_lines_wait(bv, mb, nl);
  PH(10)
  if (threadIdx.x < 4) {
    const int h = threadIdx.x;
    e0[h] = h < nl ? io[h * LSO] : 0.0;
    e1[h] = h < nl ? io[h * LSO + n2 - 1] : 0.0;
  }
  // T along the rows (ar_forward, transforms.hpp:148-160)
  const double ri = bt.rinv;
  double2* dbuf = sm + g * F::LD;
  const int N2 = bt.N;
  pk_fill<M, TD, BLUE>(dbuf, bt, t, [&](int hh, int j) {
    const int h = 2 * g + hh;
    if (h >= nl) return make_double2(0.0, 0.0);
    const double vj = io[h * LSO + j], vm = io[h * LSO + N2 - j];
    return make_double2(vj + vm, vj - vm);
  });
  PH(11)
  __shared__ double2 pfa_aux[2][2 * Pfa<M>::N1];  // prime-factor lines: u0 + Rader sums per line
  blue_core<M, TD, 2, BLUE>(sm, dbuf, bt, twd, t, pfa_aux[g]);
  PH(12)
  pk_split2<M, BLUE, LMAX>(dbuf, bt, io + (2 * g) * LSO, io + (2 * g + 1) * LSO, t, TD, pfa_aux[g]);
  __syncthreads();
  // the DST lines are free now: stage the f rows there (L2-prefetched at
  // kernel start) behind the scans
  double* fS = reinterpret_cast<double*>(sm);
  if (fimg) stage_lines(fS, LS, fimg, nl, n2);
  cp_async_commit();
  odd_scans2<LMAX>(io, LSO, 4, bt);
  cp_async_wait_all();
  if (bx && nl > 0) mbar_wait(mb + 1, 0);
  __syncthreads();
  PH(13)
  // x_k = x_{k-1} + tau * T v (solver.hpp:106), rows r0..r0+nl-1 contiguous
  double* xn = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N)) + (size_t)r0 * n2;
  const double ia = 1.0 / bt.alpha, tau = a.tau;
  double p0 = 0.0, p1 = 0.0;
  for (int h = 0; h < nl; ++h) {
    const double a0 = ia * e0[h], a1 = ia * e1[h];
    const double* o = io + h * LSO;
    double* xs = stX + h * XS + XO;
    const double* fs = fS + h * LS;
    double* xr = xn + (size_t)h * n2;
#pragma unroll 4
    for (int k = threadIdx.x; k < n2; k += NT) {
      const double t1 = (double)k * ri;
      double w = pk_at<LMAX>(o, k) + a0 * (1.0 - t1) + a1 * t1;  // o[0], o[n2-1] in bounds
      w = k == 0 ? a0 : k == n2 - 1 ? a1 : w;
      const double xv = xs[k] + tau * w;
      xr[k] = xv;
      xs[k] = xv;
      p0 += xv * xv;
      if (fimg) {
        const double e = xv - fs[k];
        p1 += e * e;
      }
    }
  }
  __syncthreads();  // x rows complete; DST buffers free for the conv lines
  PH(14)
  if constexpr (SEP) {
    // separable pipeline: row pass of A x_k as the direct row correlation of
    // the AR-extended x_k rows (work region: the f rows are consumed)
    // (the x_k rows, extended in place around offset 16)
    const int q2 = a.q2;
    for (int idx = threadIdx.x; idx < 8 * q2; idx += NT) {
      const int h = idx / (2 * q2), m = idx - h * 2 * q2;
      double* xr = stX + h * XS + XO;
      if (h < nl) {
        if (m < q2) {
          const int k = q2 - m;
          xr[-k] = 2.0 * xr[0] - xr[k];
        } else {
          const int k = m - q2 + 1;
          xr[n2 - 1 + k] = 2.0 * xr[n2 - 1] - xr[n2 - 1 - k];
        }
      }
    }
    __syncthreads();
    sep_row_pass(stX + XO - q2, XS, a.conv, q2, n2, nl, reinterpret_cast<double*>(a.zbuf) + (size_t)b * N + r0,
                 n1);
    (void)twc;
    (void)Lh;
  } else {
    const int ra = r0 + 2 * g, rb = ra + 1;
    conv_fwd_rows<L2, TD>(sm + g * F::LC, stX + (2 * g) * XS + XO, stX + (2 * g + 1) * XS + XO, n2, a.q2, twc,
                          a.zbuf + (size_t)b * n1 * Lh, ra, rb, n1, Lh, t, 1 + g);
  }
  PH(15)
  if (a.part.p) {
    double* P = a.part.p + (size_t)b * NUM_SLOTS * a.part.cap;
    const double s0 = block_sum<NT>(p0, red);
    if (threadIdx.x == 0) P[SLOT_X2 * a.part.cap + blockIdx.x] = s0;
    const double s1 = block_sum<NT>(p1, red);
    if (threadIdx.x == 0) P[SLOT_XF2 * a.part.cap + blockIdx.x] = s1;
  }
}

// ---------------------------------------------------------------------------
// rows_ainv_resid: FOUR rows per CTA, two packed conv lines of T threads each
// (T sized for the conv radices, not the DST).  The residual never leaves the
// registers: g is prefetched into registers before the inverse FFT, r = g - A x
// is written straight into the forward line at its extended position q2 + c,
// and the horizontal AR extension is filled from the line itself.
template <int L2>
struct RsCfg {
  static constexpr int T = line_threads(L2, 8), G = 2, NT = T * G;
  static constexpr int LC = padded_len(L2);
  static constexpr int LS = (L2 + 1) / 2 * 2 + 4;  // g row stride (doubles), n2 <= L2
  static constexpr size_t gs = (size_t)G * LC * 16;
  static constexpr size_t twc = gs + (size_t)4 * LS * 8;
  static constexpr size_t bytes = twc + (size_t)fft::twiddles_needed(L2) * 16;
};

template <int L2>
__global__ void __launch_bounds__(RsCfg<L2>::NT, 2) rows_ainv_resid(SpecArgs a) {
  DBX_PDL_WAIT();
  using C = RsCfg<L2>;
  constexpr int T = C::T, NT = C::NT, LS = C::LS;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double red[32];
  const double2* twc = stage_twiddles<L2, true>(reinterpret_cast<double2*>(reinterpret_cast<char*>(sm) + C::twc),
                                                a.conv.tw2);
  const int n1 = a.n1, n2 = a.n2, Lh = a.conv.Lh, q2 = a.q2;  // n2 <= L2 - 2 q2
  const size_t N = (size_t)n1 * n2;
  const int g = threadIdx.x / T, t = threadIdx.x - g * T;
  const int ra = 4 * blockIdx.x + 2 * g, rb = ra + 1;
  const bool has_a = ra < n1, has_b = rb < n1;
  double2* buf = sm + g * C::LC;
  const int bar = 1 + g;
  // g rows staged behind the inverse FFT (cp.async, rows r0..r0+3 contiguous)
  double* gS = reinterpret_cast<double*>(reinterpret_cast<char*>(sm) + C::gs);
  const int r0 = 4 * blockIdx.x, nl = n1 - r0 < 4 ? n1 - r0 : 4;
  __shared__ unsigned long long mb[1];
  bulk_init(mb, 1);
  const bool bg = stage_lines_bulk(gS, LS, a.g + (size_t)b * N + (size_t)r0 * n2, nl, n2, mb);
  cp_async_commit();
  conv_inv_load<L2, T>(buf, a.ybuf + (size_t)b * n1 * y_stride(Lh), ra, rb, n1, Lh, t);
  cp_async_wait_group<1>();  // twiddles
  __syncthreads();
  fft::fft<L2, +1, T>(buf, twc, t, bar);
  stage_lines_wait(bg, mb, nl);  // g rows visible
  // r = g - A x (solver.hpp:105) and its horizontal AR extension
  // (boundary.hpp:56-62) produced inside the forward FFT's first-stage loads
  // straight from A x (the inverse output still in the line) and the g rows
  const double* gA = gS + (2 * g) * LS;
  const double* gB = gA + LS;
  const int wext = n2 + 2 * q2;
  double p0 = 0.0;
  auto rr = [&](int c) {
    const double2 ax = buf[pad<L2>(c)];
    return make_double2(has_a ? gA[c] - ax.x : 0.0, has_b ? gB[c] - ax.y : 0.0);
  };
  fft::fft_in<L2, -1, T>(buf, twc, t, bar, [&](int p) {
    const int j = p - q2;
    int jc = j < 0 ? -j : j >= n2 ? 2 * (n2 - 1) - j : j;
    jc = jc < 0 ? 0 : jc;
    double2 v = rr(jc);
    if (j < 0 || j >= n2) {
      const double2 e = rr(j < 0 ? 0 : n2 - 1);
      v = p < wext ? make_double2(2.0 * e.x - v.x, 2.0 * e.y - v.y) : make_double2(0.0, 0.0);
    } else {
      p0 += v.x * v.x + v.y * v.y;
    }
    return v;
  });
  double2* Z = a.zbuf + (size_t)b * n1 * Lh;
  const bool pair = has_b && ((ra | n1) & 1) == 0;
  for (int k = t; k < Lh; k += T) {
    const double2 zk = buf[pad<L2>(k)], zm = buf[pad<L2>(k == 0 ? 0 : L2 - k)];
    const double2 za = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    const double2 zb = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
    if (pair) {
      st_pair(Z + (size_t)k * n1 + ra, za, zb);
    } else {
      if (has_a) Z[(size_t)k * n1 + ra] = za;
      if (has_b) Z[(size_t)k * n1 + rb] = zb;
    }
  }
  if (a.part.p) {
    double* P = a.part.p + (size_t)b * NUM_SLOTS * a.part.cap;
    const double s0 = block_sum<NT>(p0, red);
    if (threadIdx.x == 0) P[SLOT_R2 * a.part.cap + blockIdx.x] = s0;
  }
  if (a.fin_cnt) finalize_last_block(a.fin, a.fin_cnt, b);
}

// ---------------------------------------------------------------------------
// rows_resid_sep (separable pipeline): FOUR rows per CTA.  r = g - A x_k
// (A x_k rows from the column pass, row-major in ybuf; a.in == nullptr: r = g,
// the first A' of a run) with ||r||^2 partials, then the row pass of A' r: the
// AR-extended r rows correlated with the A' row taps -> Z'^T (solver.hpp:105,
// blur.hpp:75-90 restricted to one axis).
constexpr int kResidNT = 256;

__host__ __device__ constexpr int resid_ls(int n2) { return (n2 + 1) / 2 * 2 + 4; }
// g / r rows: data at offset 16 (128-byte aligned for the bulk copy), the 2 q2
// AR extension samples written around them in place, stride = 4 mod 16
__host__ __device__ constexpr int resid_lsr(int n2, int q2) {
  const int e = 16 + n2 + q2 + 9;
  return e + ((4 - e % 16) + 16) % 16;
}
// only the g / r rows are staged: A x is read straight from global in the
// residual loop (coalesced, once), halving the shared memory per CTA so four
// CTAs fit per SM
__host__ __device__ constexpr size_t resid_sep_bytes(int n2, int q2) {
  return (size_t)4 * resid_lsr(n2, q2) * 8;
}

__global__ void __launch_bounds__(kResidNT, 4) rows_resid_sep(SpecArgs a) {
  DBX_PDL_WAIT();
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double red[32];
  __shared__ unsigned long long mb[1];
  const int n1 = a.n1, n2 = a.n2, q2 = a.q2, LSR = resid_lsr(n2, q2);
  const size_t N = (size_t)n1 * n2;
  const int r0 = 4 * blockIdx.x, nl = n1 - r0 < 4 ? n1 - r0 : 4;
  double* rS = reinterpret_cast<double*>(sm);  // g rows at offset 16, then r in place + extension
  const bool have_y = a.in != nullptr;
  bulk_init(mb, 1);
  const bool bg = stage_lines_bulk(rS + 16, LSR, a.g + (size_t)b * N + (size_t)r0 * n2, nl, n2, mb);
  cp_async_commit();
  // A x rows into registers while g lands (8 per thread at n2 = 1024)
  constexpr int YR = 8;
  const double* yg = have_y ? a.in + (size_t)b * N + (size_t)r0 * n2 : nullptr;
  const int tot = nl * n2;
  double yv[YR];
#pragma unroll
  for (int k = 0; k < YR; ++k) {
    const int e = threadIdx.x + k * kResidNT;
    yv[k] = have_y && e < tot ? __ldcs(yg + e) : 0.0;
  }
  cp_async_wait_all();
  __syncthreads();
  stage_lines_wait(bg, mb, nl);
  double p0 = 0.0;
#pragma unroll
  for (int k = 0; k < YR; ++k) {
    const int e = threadIdx.x + k * kResidNT;
    if (e < tot) {
      const int h = e / n2, c = e - h * n2;
      double* rr = rS + h * LSR + 16;
      const double rv = rr[c] - yv[k];
      rr[c] = rv;
      p0 += rv * rv;
    }
  }
  for (int e = threadIdx.x + YR * kResidNT; e < tot; e += kResidNT) {
    const int h = e / n2, c = e - h * n2;
    double* rr = rS + h * LSR + 16;
    const double rv = have_y ? rr[c] - __ldcs(yg + e) : rr[c];
    rr[c] = rv;
    p0 += rv * rv;
  }
  __syncthreads();
  // horizontal AR extension of the r rows in place (boundary.hpp:56-62)
  for (int idx = threadIdx.x; idx < 8 * q2; idx += kResidNT) {
    const int h = idx / (2 * q2), m = idx - h * 2 * q2;
    double* rr = rS + h * LSR + 16;
    if (h < nl) {
      if (m < q2) {
        const int k = q2 - m;
        rr[-k] = 2.0 * rr[0] - rr[k];
      } else {
        const int k = m - q2 + 1;
        rr[n2 - 1 + k] = 2.0 * rr[n2 - 1] - rr[n2 - 1 - k];
      }
    }
  }
  __syncthreads();
  sep_row_pass(rS + 16 - q2, LSR, a.conv, q2, n2, nl, reinterpret_cast<double*>(a.zbuf) + (size_t)b * N + r0, n1);
  if (a.part.p) {
    double* P = a.part.p + (size_t)b * NUM_SLOTS * a.part.cap;
    const double s0 = block_sum<kResidNT>(p0, red);
    if (threadIdx.x == 0) P[SLOT_R2 * a.part.cap + blockIdx.x] = s0;
  }
  if (a.fin_cnt) finalize_last_block(a.fin, a.fin_cnt, b);
}

// ---------------------------------------------------------------------------
// Column half of D on the transposed intermediate: line c of u^T (column c of
// u) is contiguous.  T~ -> multiply by d^T[c][.] -> T, result written into the
// row-major s.  FOUR adjacent columns per CTA, two per packed complex DFT
// (pk_fill / pk_split), so the row-major stores are full 32-byte sectors.
template <int M, bool BLUE>
struct TcolSmem {
  static constexpr int TD = fused_td(M);
  static constexpr int LMAX = BLUE ? M / 2 + 1 : M + 1;         // max line length n
  static constexpr int LS = (LMAX + 1) / 2 * 2 + 4;             // line stride (doubles): 4 lines hit distinct banks
  static constexpr int LSO = ((LMAX > PkOut<LMAX>::OL ? LMAX : PkOut<LMAX>::OL) + 1) / 2 * 2 + 4;  // io lines
  static constexpr size_t off_io = (size_t)2 * padded_len(M) * 16;
  static constexpr size_t off_d = off_io + (size_t)4 * LSO * 8;
  // DL (DBX_TC_MINB >= 3): d^T is not staged — it multiplies the T~ outputs in
  // place straight from global (L2-resident, shared by the batch) — and the
  // twiddles are read through L1, so three CTAs fit per SM
  static constexpr bool DL = DBX_TC_MINB >= 3;
  static constexpr size_t off_tw = off_d + (DL ? 0 : (size_t)4 * LS * 8);
  static constexpr size_t TWB = (size_t)dst_twiddles_needed(M) * 16;
  static constexpr bool TW = !DL && off_tw + TWB <= 115200;  // keep 2 CTAs / SM
  static constexpr size_t bytes = TW ? off_tw + TWB : off_tw;
};

template <int M, bool BLUE>
__global__ void __launch_bounds__(2 * fused_td(M), DBX_TC_MINB) dst_tcols(SpecArgs a) {
  DBX_PDL_WAIT();
  using S = TcolSmem<M, BLUE>;
  constexpr int TD = S::TD, NT = 2 * TD, LS = S::LS, LSO = S::LSO, LMAX = S::LMAX;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double e0[4], e1[4];
  char* base = reinterpret_cast<char*>(sm);
  double* io = reinterpret_cast<double*>(base + S::off_io);  // 4 lines: input, then DST outputs
  double* dS = reinterpret_cast<double*>(base + S::off_d);   // 4 d^T lines
  const BlueTables& bt = a.blue1;
  const double2* tw = stage_twiddles<M, S::TW>(reinterpret_cast<double2*>(base + S::off_tw), bt.tw);
  const int n = a.n1, n2 = a.n2;
  const size_t N = (size_t)n * n2;
  PH_DECL
  const int c0 = 4 * blockIdx.x;
  const int nl = n2 - c0 < 4 ? n2 - c0 : 4;
  __shared__ unsigned long long mb[2];
  bulk_init(mb, 2);
  const bool bi = stage_lines_bulk(io, LSO, a.in + (size_t)b * N + (size_t)c0 * n, nl, n, mb);  // u^T lines
  cp_async_commit();
  const double* dg = a.dT + (size_t)b * a.dstride + (size_t)c0 * n;
  const bool bd = S::DL ? false : stage_lines_bulk(dS, LS, dg, nl, n, mb + 1);  // d^T
  cp_async_commit();
  cp_async_wait_group<1>();
  __syncthreads();
  stage_lines_wait(bi, mb, nl);
  PH(0)
  if (threadIdx.x < 4) {
    const int h = threadIdx.x;
    e0[h] = h < nl ? io[h * LSO] : 0.0;
    e1[h] = h < nl ? io[h * LSO + n - 1] : 0.0;
  }
  const int g = threadIdx.x / TD, t = threadIdx.x - g * TD;
  double2* buf = sm + g * padded_len(M);
  const double ri = bt.rinv;
  // T~ (ar_inverse, transforms.hpp:163-173) of lines 2g, 2g+1
  const int NL = bt.N;
  const double xa0 = io[(2 * g) * LSO], xae = io[(2 * g) * LSO + n - 1];
  const double xb0 = io[(2 * g + 1) * LSO], xbe = io[(2 * g + 1) * LSO + n - 1];
  pk_fill<M, TD, BLUE>(buf, bt, t, [&](int hh, int j) {
    const int h = 2 * g + hh;
    if (h >= nl) return make_double2(0.0, 0.0);
    const double* L = io + h * LSO;
    const double x0 = hh ? xb0 : xa0, xe = hh ? xbe : xae;
    const double lj = L[j], lm = L[NL - j];
    return make_double2(lj + lm - (x0 + xe), (lj - lm) - (x0 - xe) * fma(-2.0 * ri, (double)j, 1.0));
  });
  PH(1)
  __shared__ double2 pfa_aux[2][2 * Pfa<M>::N1];  // prime-factor lines: u0 + Rader sums per line
  blue_core<M, TD, 2, BLUE>(sm, buf, bt, tw, t, pfa_aux[g]);
  PH(2)
  pk_split2<M, BLUE, LMAX>(buf, bt, io + (2 * g) * LSO, io + (2 * g + 1) * LSO, t, TD, pfa_aux[g]);
  __syncthreads();
  PH(3)
  odd_scans2<LMAX>(io, LSO, 4, bt);
  cp_async_wait_all();
  if (bd && nl > 0) mbar_wait(mb + 1, 0);
  __syncthreads();
  __shared__ double dd0[4], dd1[4];
  if constexpr (S::DL) {
    // u o d in place on the T~ outputs (pk_at layout), d^T from global,
    // four loads in flight per thread
    using P = PkOut<LMAX>;
    constexpr int U = 4;
    for (int e0i = threadIdx.x; e0i < nl * n; e0i += U * NT) {
      double dv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0i + u * NT;
        dv[u] = e < nl * n ? __ldg(dg + (e / n) * n + (e - (e / n) * n)) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int e = e0i + u * NT;
        if (e < nl * n) {
          const int h = e / n, k = e - h * n, m = k >> 1;
          double* o = io + h * LSO + ((k & 1) ? P::EB + (m & 15) * P::STR1 + (m >> 4) : m);
          *o *= dv[u];
          if (k == 0) dd0[h] = dv[u];
          if (k == n - 1) dd1[h] = dv[u];
        }
      }
    }
    __syncthreads();
  }
  PH(4)
  // v = u o d (u_0 = alpha v_0, u_{n-1} = alpha v_{n-1}), then T (ar_forward)
  pk_fill<M, TD, BLUE>(buf, bt, t, [&](int hh, int j) {
    const int h = 2 * g + hh;
    if (h >= nl) return make_double2(0.0, 0.0);
    const double* o = io + h * LSO;
    if constexpr (S::DL) {
      const double mj = pk_at<LMAX>(o, j), mm = pk_at<LMAX>(o, NL - j);
      return make_double2(mj + mm, mj - mm);
    } else {
      const double mj = pk_at<LMAX>(o, j) * dS[h * LS + j], mm = pk_at<LMAX>(o, NL - j) * dS[h * LS + NL - j];
      return make_double2(mj + mm, mj - mm);
    }
  });
  PH(5)
  blue_core<M, TD, 2, BLUE>(sm, buf, bt, tw, t, pfa_aux[g]);
  PH(6)
  pk_split2<M, BLUE, LMAX>(buf, bt, io + (2 * g) * LSO, io + (2 * g + 1) * LSO, t, TD, pfa_aux[g]);
  __syncthreads();
  PH(7)
  odd_scans2<LMAX>(io, LSO, 4, bt);
  __syncthreads();
  PH(8)
  // T output w_0 = v_0 / alpha = e0 d_0, w_{n-1} = e1 d_{n-1}, interior DST + ramp
  // (NT % 4 == 0: each thread keeps one column h; 4 threads fill a 32-byte sector)
  static_assert(NT % 4 == 0, "column-group mapping");
  const int h = threadIdx.x & 3;
  if (h < nl) {
    double* s = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N)) + c0 + h;
    const double* o = io + h * LSO;
    const double a0 = e0[h] * (S::DL ? dd0[h] : dS[h * LS]), a1 = e1[h] * (S::DL ? dd1[h] : dS[h * LS + n - 1]);
#pragma unroll 4
    for (int k = threadIdx.x >> 2; k < n; k += NT / 4) {
      const double t1 = (double)k * ri;
      const double w = pk_at<LMAX>(o, k) + a0 * (1.0 - t1) + a1 * t1;  // o[0], o[n-1] in bounds
      s[(size_t)k * n2] = k == 0 ? a0 : k == n - 1 ? a1 : w;
    }
  }
  PH(9)
}

// WHICH makes the attribute flag per kernel (the three kernels share one
// function-pointer type).
template <int L2, int M, bool BLUE, int WHICH, typename K>
int fused_launch(K kernel, const SpecArgs& a, cudaStream_t s) {
  using F = Fused<L2, M, BLUE>;
  // WHICH: 0 tt, 1 t_axpy, 2 resid, 4 tt (separable), 5 t_axpy (separable)
  constexpr size_t bytes = WHICH == 0 ? F::tt_bytes : WHICH == 4 ? F::tts_bytes
                           : (WHICH == 1 || WHICH == 5) ? F::ax_bytes : RsCfg<L2>::bytes;
  constexpr int nt = WHICH == 2 ? RsCfg<L2>::NT : F::NT;
  constexpr int rows = 4;  // rows per CTA
  static AttrOnce attr;
  if (!attr.ensure(kernel, bytes)) return -1;
  dim3 grid((a.n1 + rows - 1) / rows, a.batch);
  launch_k(kernel, grid, nt, bytes, s, a);
  return (int)grid.x;
}

template <int M, bool BLUE>
int tcols_launch(const SpecArgs& a, cudaStream_t s) {
  using SMP = TcolSmem<M, BLUE>;
  static AttrOnce attr;
  if (!attr.ensure(dst_tcols<M, BLUE>, SMP::bytes)) return -1;
  dim3 grid((a.n2 + 3) / 4, a.batch);
  launch_k(dst_tcols<M, BLUE>, grid, 2 * SMP::TD, SMP::bytes, s, a);
  return (int)grid.x;
}

}  // namespace

#ifdef DBX_PHASES
int fused_debug_phases(unsigned long long* out, int n) {
  if (n > 64) n = 64;
  cudaDeviceSynchronize();
  if (cudaMemcpyFromSymbol(out, g_phase, n * sizeof(unsigned long long)) != cudaSuccess) return -1;
  static const unsigned long long zero[64] = {};
  cudaMemcpyToSymbol(g_phase, zero, sizeof zero);
  return n;
}
#endif

// (conv L2, DST M, Bluestein?) combinations compiled for the fused pipeline.
#define DBX_FUSED_LIST(X) X(1080, 1023, false) X(540, 1024, true) X(540, 511, false) X(270, 255, false)

bool fused_sep_supported(int L2, int M, bool blue, int n2, int q2) {
  if (!conv_sep_supported(q2) || resid_sep_bytes(n2, q2) > 200 * 1024) return false;
#define X(L, MM, BL) \
  if (L2 == (L) && M == (MM) && blue == (BL)) return n2 <= Fused<L, MM, BL>::LMAX && q2 <= 15;
  DBX_FUSED_LIST(X)
#undef X
  return false;
}

bool fused_supported(int L2, int M, bool blue) {
#define X(L, MM, BL) if (L2 == (L) && M == (MM) && blue == (BL)) return Fused<L, MM, BL>::ax_bytes <= 200 * 1024 && TcolSmem<MM, BL>::bytes <= 200 * 1024;
  DBX_FUSED_LIST(X)
#undef X
  return false;
}

int launch_fused(int which, const SpecArgs& a, cudaStream_t s) {
  if (which == FUSED_RESID_SEP) {
    const size_t bytes = resid_sep_bytes(a.n2, a.q2);
    if (!set_smem(rows_resid_sep, bytes)) return -1;
    dim3 grid((a.n1 + 3) / 4, a.batch);
    launch_k(rows_resid_sep, grid, kResidNT, bytes, s, a);
    return (int)grid.x;
  }
  // warp-owned column half (wdst.cu) for 1024-point columns; DBX_WDST=0
  // keeps the CTA lock-step dst_tcols (A/B and tests)
  static const bool wdst_off = [] { const char* e = getenv("DBX_WDST"); return e && e[0] == '0'; }();
  if (which == FUSED_DST_TCOLS && !wdst_off) {
    const int c = launch_dst_tcols_w(a, s);
    if (c >= 0) return c;
  }
  // warp-owned separable row kernels (wdst.cu) for 1024-point rows;
  // DBX_WROWS=0 keeps the CTA lock-step ones (A/B and tests)
  // (DBX_WROWS=2: rows_tt_w only, 3: rows_t_axpy_w only)
  static const int wrows = [] { const char* e = getenv("DBX_WROWS"); return e ? atoi(e) : 1; }();
  if ((which == FUSED_TT_SEP && (wrows == 1 || wrows == 2)) || (which == FUSED_T_AXPY_SEP && (wrows == 1 || wrows == 3))) {
    const int c = launch_rows_w(which == FUSED_TT_SEP ? 0 : 1, a, s);
    if (c >= 0) return c;
  }
  const int L2 = a.conv.L2, M = a.blue2.M;
  const bool blue = a.blue2.M != a.blue2.N;
#define X(L, MM, BL)                                                                          \
  if (L2 == (L) && M == (MM) && blue == (BL)) {                                               \
    if (which == FUSED_AINV_TT) return fused_launch<L, MM, BL, 0>(rows_ainv_tt<L, MM, BL>, a, s); \
    if (which == FUSED_T_AXPY_AFWD) return fused_launch<L, MM, BL, 1>(rows_t_axpy_afwd<L, MM, BL>, a, s); \
    if (which == FUSED_AINV_RESID) return fused_launch<L, MM, BL, 2>(rows_ainv_resid<L>, a, s); \
    if (which == FUSED_DST_TCOLS) return tcols_launch<MM, BL>(a, s);                             \
    if (which == FUSED_TT_SEP) return fused_launch<L, MM, BL, 4>(rows_ainv_tt<L, MM, BL, true>, a, s); \
    if (which == FUSED_T_AXPY_SEP) return fused_launch<L, MM, BL, 5>(rows_t_axpy_afwd<L, MM, BL, true>, a, s); \
  }
  DBX_FUSED_LIST(X)
#undef X
  return -1;
}

}  // namespace dbx
