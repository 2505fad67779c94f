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

#include <cstdlib>

#include "spectral_common.cuh"

namespace dbx {


namespace {

template <int L2>
__global__ void __launch_bounds__(lines_for(L2, kConvBudget, 8) * line_threads(L2, 8), conv_row_minb(L2))
conv_row_fwd(SpecArgs a) {
  DBX_PDL_WAIT();
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
      if (ra < n1) va[i] = hext(x, ra, j, n2, a.bc);
      if (rb < n1) vb[i] = hext(x, rb, j, n2, a.bc);
    }
  }
#pragma unroll
  for (int i = 0; i < PF; ++i) {
    const int p = t + i * T;
    if (p < L2) buf[pad<L2>(p)] = make_double2(va[i], vb[i]);
  }
  cp_async_wait_all();
  __syncthreads();
  fft::fft<L2, -1, T>(buf, tw, t, G > 1 ? 1 + g : 0);
  double2* Z = a.zbuf + (size_t)b * n1 * Lh;
  // ztrans: spectra stored [k][row] so the column pass reads contiguously;
  // the pair's two rows are adjacent (one 32-byte sector per k)
  const size_t sr = a.ztrans ? 1 : (size_t)Lh, sk = a.ztrans ? (size_t)n1 : 1;
  for (int k = t; k < Lh; k += T) {
    const double2 zk = buf[pad<L2>(k)], zm = buf[pad<L2>(k == 0 ? 0 : L2 - k)];
    if (ra < n1) Z[ra * sr + k * sk] = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
    if (rb < n1) Z[rb * sr + k * sk] = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
  }
}

template <int L1>
__global__ void __launch_bounds__(lines_for(L1, kConvBudget, 8) * line_threads(L1, 8))
conv_col(SpecArgs a) {
  DBX_PDL_WAIT();
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
  // cp.async groups: twiddles, (ztrans) this line's spectrum column, then the
  // kernel-spectrum columns ([k2][k1] layout, contiguous in p) which may still
  // be in flight during the forward FFT
  double2* hst = sm + SM::lines + g * padded_len(L1);
  const double2* tw = stage_twiddles<L1, SM::TW>(sm + SM::lines + (SM::HS ? SM::lines : 0), a.conv.tw1);
  const double2* Hcol = a.conv.H + (size_t)(kk < Lh ? kk : 0) * L1;
  const double2* Z = a.zbuf + (size_t)b * n1 * Lh;
  const int hext_rows = n1 + 2 * q1;
  double2* buf = sm + g * padded_len(L1);
  if (a.ztrans) {
    // column kk of Z^T is contiguous: copy it straight into rows q1 .. q1+n1-1
    // of the line (no registers, all loads in flight at once)
    if (kk < Lh) {
      const double2* zc = Z + (size_t)kk * n1;
      for (int rho = t; rho < n1; rho += T) cp_async16(buf + pad<L1>(rho + q1), zc + rho);
    }
    cp_async_commit();
    // bulk-prefetch into L2 the column of the CTA one resident wave ahead, so
    // its copies hit L2 instead of waiting on HBM
    if (t == 0) {
      const long long ahead = (long long)blockIdx.y * gridDim.x + blockIdx.x + 2 * nsm();
      const int bb = (int)(ahead / gridDim.x), kx = (int)(ahead % gridDim.x) * G + g;
      if (bb < a.batch && kx < Lh)
        prefetch_l2(a.zbuf + (size_t)bb * n1 * Lh + (size_t)kx * n1, (unsigned)n1 * 16);
    }
    if constexpr (SM::HS) {
      for (int p = t; p < L1; p += T) cp_async16(hst + p, Hcol + p);
    }
    cp_async_commit();
    cp_async_wait_group<1>();
    __syncthreads();
    // vertical AR extension synthesised spectrally (Z[-i] = 2 Z[0] - Z[i]) and
    // the zero tail, from the rows already in shared memory
    for (int p = t; p < L1; p += T) {
      if (p >= q1 && p < q1 + n1) continue;
      double2 v = make_double2(0.0, 0.0);
      if (kk < Lh && p < hext_rows) {
        const int rho = p - q1;
        if (a.bc == DBX_BC_REFLECTIVE) {
          v = buf[pad<L1>((rho < 0 ? -rho - 1 : 2 * n1 - 1 - rho) + q1)];
        } else {
          const int r0 = rho < 0 ? 0 : n1 - 1, ri = rho < 0 ? -rho : 2 * (n1 - 1) - rho;
          const double2 z0 = buf[pad<L1>(r0 + q1)], zi = buf[pad<L1>(ri + q1)];
          v = make_double2(2.0 * z0.x - zi.x, 2.0 * z0.y - zi.y);
        }
      }
      buf[pad<L1>(p)] = v;
    }
    if (kk >= Lh)
      for (int p = q1 + t; p < q1 + n1; p += T) buf[pad<L1>(p)] = make_double2(0.0, 0.0);
    __syncthreads();
  } else {
    if constexpr (SM::HS) {
      for (int p = t; p < L1; p += T) cp_async16(hst + p, Hcol + p);
    }
    cp_async_commit();
    cp_async_commit();  // (empty) keeps the group count of the ztrans branch
    // load the G columns with the vertical AR extension synthesised spectrally
    // (loads batched in registers first, then stored)
    constexpr int PF = (L1 * G + NT - 1) / NT;
    double2 v[PF];
#pragma unroll
    for (int i = 0; i < PF; ++i) {
      const int idx = threadIdx.x + i * NT;
      const int p = idx / G, gg = idx - p * G;
      const int k = k0 + gg;
      v[i] = make_double2(0.0, 0.0);
      if (idx < L1 * G && k < Lh && p < hext_rows && a.preext) {
        v[i] = Z[(size_t)p * Lh + k];  // row slab: halo / global AR rows supplied by the caller
      } else if (idx < L1 * G && k < Lh && p < hext_rows) {
        const int rho = p - q1;
        if (a.bc == DBX_BC_REFLECTIVE && (rho < 0 || rho >= n1)) {
          // reflective rows are copies: Z[-i] = Z[i-1], Z[n-1+i] = Z[n-i]
          v[i] = Z[(size_t)(rho < 0 ? -rho - 1 : 2 * n1 - 1 - rho) * Lh + k];
        } else if (rho < 0) {
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
    cp_async_wait_group<2>();  // twiddles landed (H may still be in flight)
    __syncthreads();
  }
  const int bar = G > 1 ? 1 + g : 0;
  if constexpr (kConvCt) {
    // cyclic convolution in place: DIF -> x digit-reversed spectrum -> DIT
    static_assert(fft::ct_twiddles_needed(L1) <= fft::twiddles_needed(L1), "CT twiddle prefix");
    if constexpr (SM::HS) {
      cp_async_wait_all();
      fft::line_sync(bar, T);  // the line's H entries (staged by all its threads) visible
    }
    fft::ct_convolve<L1, T>(buf, tw, SM::HS ? hst : Hcol, t, bar, nullptr);
  } else {
  fft::fft<L1, -1, T>(buf, tw, t, bar);
  // the kernel-spectrum product rides on the inverse FFT's first-stage loads
  if constexpr (SM::HS) {
    cp_async_wait_all();
    fft::line_sync(bar, T);  // the line's H entries (staged by all its threads) visible
    fft::fft_in<L1, +1, T>(buf, tw, t, bar, [&](int p) { return cmul(buf[pad<L1>(p)], hst[p]); });
  } else {
    fft::fft_in<L1, +1, T>(buf, tw, t, bar, [&](int p) { return cmul(buf[pad<L1>(p)], __ldg(Hcol + p)); });
  }
  }
  if (G > 1) __syncthreads();  // the stores interleave the CTA's lines
  const int YS = y_stride(Lh);
  double2* Y = a.ybuf + (size_t)b * n1 * YS;
  if (G == 2 && k0 + 1 < Lh) {
    // the CTA's two adjacent columns of one row: one 32-byte store
    for (int p = threadIdx.x; p < n1; p += NT)
      st_pair(Y + (size_t)p * YS + k0, sm[pad<L1>(p)], sm[padded_len(L1) + pad<L1>(p)]);
  } else {
    for (int idx = threadIdx.x; idx < n1 * G; idx += NT) {
      const int p = idx / G, gg = idx - p * G, k = k0 + gg;
      if (k < Lh) Y[(size_t)p * YS + k] = sm[gg * padded_len(L1) + pad<L1>(p)];
    }
  }
}

template <int L2>
__global__ void __launch_bounds__(lines_for(L2, kConvBudget, 8) * line_threads(L2, 8), conv_row_minb(L2))
conv_row_inv(SpecArgs a) {
  DBX_PDL_WAIT();
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
  const double2* Y = a.ybuf + (size_t)b * n1 * y_stride(Lh);
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
      if (ra < n1) A[i] = Y[(size_t)ra * y_stride(Lh) + k];
      if (rb < n1) Bv[i] = Y[(size_t)rb * y_stride(Lh) + k];
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
  fft::fft<L2, +1, T>(buf, tw, t, G > 1 ? 1 + g : 0);
  // operand loads (g / x_{k-1} / f / d) four deep per thread (epi_row)
  if (ra < n1) epi_row<4>(e, (size_t)ra * n2, n2, t, T, [&](int c) { return buf[pad<L2>(c)].x; });
  if (rb < n1) epi_row<4>(e, (size_t)rb * n2, n2, t, T, [&](int c) { return buf[pad<L2>(c)].y; });
  write_partials<NT>(a, e, red, b);
}

// ---------------------------------------------------------------------------
// Column pass of a RANK-1 mask, w(t,u) = a_t b_u (the axis-aligned Gaussians of
// C1, C3, C5).  The kernel spectrum factors, H[k2][k1] = conj(A(k1)) conj(B(k2))
// / (L1 L2), so FFT_L1 -> x H -> IFFT_L1 of column k2 is the valid direct
// correlation of the vertically AR-extended column with a, times
// beta(k2) = conj(B(k2)) / L2:  Y[i][k2] = beta(k2) sum_t a_t Zext[i + t][k2]
// (boundary.hpp:56-64 extension, blur.hpp:39-52 correlation along one axis).
// 2q1+1 complex-by-real FMA pairs per output instead of two L1-point FFTs: no
// barriers inside the arithmetic, every thread an independent register-blocked
// stencil.  CK = 4 adjacent columns per CTA in a skewed smem layout (element p
// of a column at p + p/8): lane (j, c) of a warp reads rows 8m + s of column c,
// so each 8-lane phase hits 8 distinct 16-byte bank groups, and the stores of a
// row's 4 columns are 64 contiguous bytes.
constexpr int kSepCK = 4, kSepR = 8, kSepNT = 256, kSepBand = 1024;

// Output rows are split into gridDim.z bands of sep_band rows (a multiple of
// 8, at most kSepBand) so a CTA's staged columns stay within ~110 KB (two CTAs
// per SM) at any image height; band z stages extended rows
// [z RB, z RB + RB + 2 q1).
__host__ __device__ constexpr int sep_bands(int n1) { return (n1 + kSepBand - 1) / kSepBand; }
__host__ __device__ constexpr int sep_band(int n1, int nb) { return ((n1 + nb - 1) / nb + kSepR - 1) / kSepR * kSepR; }
__host__ __device__ constexpr int sep_stride(int rb, int q1) {
  const int e = rb + 2 * q1;
  const int s = e + e / 8 + 1;
  return s + ((2 - s % 8) + 8) % 8;  // = 2 mod 8: the 4 columns' bank groups interleave
}
__device__ __forceinline__ int skew(int p) { return p + (p >> 3); }

template <int Q>
__global__ void __launch_bounds__(kSepNT, 2) conv_col_sep(SpecArgs a) {
  DBX_PDL_WAIT();
  constexpr int NTAP = 2 * Q + 1, R = kSepR, CK = kSepCK;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  const int n1 = a.n1, Lh = a.conv.Lh;
  const int k0 = blockIdx.x * CK;
  const int RB = sep_band(n1, gridDim.z), S = sep_stride(RB, Q);
  const int p0 = blockIdx.z * RB;                     // first extended row of the band
  const int rows = min(RB, n1 - p0);                  // output rows of the band
  const int NL = RB + 2 * Q;                          // staged rows (local l = p - p0)
  const int E = n1 + 2 * Q;                           // extended column length
  const double2* Z = a.zbuf + (size_t)b * n1 * Lh;
  // ---- stage the band's staged-from-memory rows [lo, hi) (local index) with
  // cp.async: the interior rows rho = l + p0 - q1 in [0, n1), or every row
  // of the caller-extended slab (preext) ----
  int lo, hi;
  if (a.preext) {
    lo = 0;
    hi = min(NL, E - p0);
    for (int idx = threadIdx.x; idx < (hi - lo) * CK; idx += kSepNT) {
      const int l = idx / CK, c = idx % CK, k = k0 + c;
      if (k < Lh) cp_async16(sm + c * S + skew(l), Z + (size_t)(p0 + l) * Lh + k);
    }
  } else {
    const int rlo = max(0, p0 - Q), rhi = min(n1, p0 + NL - Q);
    lo = rlo + Q - p0;
    hi = rhi + Q - p0;
    if (a.ztrans) {  // column k of Z^T is contiguous in rho
      for (int c = 0; c < CK; ++c) {
        const int k = k0 + c;
        if (k >= Lh) break;
        const double2* zc = Z + (size_t)k * n1;
        for (int rho = rlo + threadIdx.x; rho < rhi; rho += kSepNT)
          cp_async16(sm + c * S + skew(rho + Q - p0), zc + rho);
      }
    } else {  // row-major spectra: the CK columns of a row are contiguous
      for (int idx = threadIdx.x; idx < (rhi - rlo) * CK; idx += kSepNT) {
        const int rho = rlo + idx / CK, c = idx % CK, k = k0 + c;
        if (k < Lh) cp_async16(sm + c * S + skew(rho + Q - p0), Z + (size_t)rho * Lh + k);
      }
    }
  }
  cp_async_commit();
  double tap[NTAP];
#pragma unroll
  for (int t = 0; t < NTAP; ++t) tap[t] = __ldg(a.conv.sepa + t);
  cp_async_wait_all();
  __syncthreads();
  // ---- the other local rows [0, lo) and [hi, NL): vertical extension (AR:
  // Z[-i] = 2 Z[0] - Z[i]; reflective copies) from staged rows, zeros past
  // the extended column ----
  for (int idx = threadIdx.x; idx < (lo + NL - hi) * CK; idx += kSepNT) {
    const int e = idx / CK, c = idx % CK, k = k0 + c;
    const int l = e < lo ? e : hi + (e - lo), p = p0 + l, rho = p - Q;
    double2 v = make_double2(0.0, 0.0);
    if (k < Lh && p < E && !a.preext) {
      const double2* col = sm + c * S;
      if (a.bc == DBX_BC_REFLECTIVE) {
        v = col[skew((rho < 0 ? -rho - 1 : 2 * n1 - 1 - rho) + Q - p0)];
      } else {
        const int r0 = rho < 0 ? 0 : n1 - 1, ri = rho < 0 ? -rho : 2 * (n1 - 1) - rho;
        const double2 z0 = col[skew(r0 + Q - p0)], zi = col[skew(ri + Q - p0)];
        v = make_double2(2.0 * z0.x - zi.x, 2.0 * z0.y - zi.y);
      }
    }
    sm[c * S + skew(l)] = v;  // reads touch staged rows only
  }
  if (k0 + CK > Lh) {  // columns past Lh: read by the stencil, never stored
    for (int idx = threadIdx.x; idx < (hi - lo) * CK; idx += kSepNT) {
      const int l = lo + idx / CK, c = idx % CK;
      if (k0 + c >= Lh) sm[c * S + skew(l)] = make_double2(0.0, 0.0);
    }
  }
  __syncthreads();
  // ---- register-blocked stencil: lane (j, c) computes rows 8m .. 8m+7 of
  // column c (m = 8 w + j + 64 it); every staged value feeds all the
  // accumulators it belongs to as soon as it is loaded ----
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int j = lane >> 2, c = lane & 3, k = k0 + c;
  const double2 beta = k < Lh ? __ldg(a.conv.sepb + k) : make_double2(0.0, 0.0);
  const int YS = y_stride(Lh);
  double2* Y = a.ybuf + (size_t)b * n1 * YS + (size_t)p0 * YS;
  const int nblk = (rows + R - 1) / R;
  for (int m = w * 8 + j; m < nblk; m += (kSepNT / 32) * 8) {
    const int i0 = m * R;
    const double2* col = sm + c * S + 9 * (i0 >> 3);  // skew(i0 + s) = 9 i0/8 + s + s/8
    double2 acc[R];
#pragma unroll
    for (int r = 0; r < R; ++r) acc[r] = make_double2(0.0, 0.0);
#pragma unroll
    for (int s = 0; s < R + 2 * Q; ++s) {
      const double2 z = col[s + (s >> 3)];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        const int t = s - r;
        if (t >= 0 && t < NTAP) {
          acc[r].x = fma(tap[t], z.x, acc[r].x);
          acc[r].y = fma(tap[t], z.y, acc[r].y);
        }
      }
    }
    if (k < Lh) {
#pragma unroll
      for (int r = 0; r < R; ++r)
        if (i0 + r < rows) Y[(size_t)(i0 + r) * YS + k] = cmul(acc[r], beta);
    }
  }
}

// ---------------------------------------------------------------------------
// Column pass of the separable (rank-1 mask) fused pipeline on REAL data:
// Y[i][c] = sum_t a_t Zext[i + t][c], Z^T = the row-correlated image stored
// transposed ([c][row], real), Zext its vertical AR extension
// (boundary.hpp:56-64), Y row-major.  CTA tile: 32 columns x a band of BAND
// rows; staged as [row][33] so a warp's lanes read 32 consecutive doubles (one
// column each) and store 256 contiguous bytes of a Y row.  Each thread: 16
// consecutive rows of its column, every staged value feeding all its
// accumulators at once (31 FMAs per output for q1 = 15).  The taps travel as
// kernel parameters: the DFMAs read them from the constant bank, so they cost
// no registers (64 fewer than taps held in registers) and more CTAs fit per SM.
constexpr int kColW = 32, kColLD = 33, kColRT = 16, kColNT = 256;

template <int NTAP>
struct ColTaps {
  double t[NTAP];
};

__host__ __device__ constexpr int col_minb(int band) { return band <= 128 ? 4 : band <= 192 ? 3 : 2; }

// MODE 0: Y -> a.ybuf (separable fused pipeline); MODE 1: Y -> a.out
// (BLUR_STORE); MODE 2: r = g - Y -> a.out with ||r||^2 partials (BLUR_RESID)
// — the separate-pass path's direct separable blur (rows_sep_seg + this).
template <int Q, int BAND, int MODE>
__global__ void __launch_bounds__(kColNT, col_minb(BAND)) cols_sep_real(SpecArgs a, const ColTaps<2 * Q + 1> tp) {
  DBX_PDL_WAIT();
  constexpr int NTAP = 2 * Q + 1, NL = BAND + 2 * Q, RT = kColRT;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double smd[];
  const int n1 = a.n1, n2 = a.n2;
  const size_t N = (size_t)n1 * n2;
  const int c0 = blockIdx.x * kColW, p0 = blockIdx.z * BAND;
  const int rows = min(BAND, n1 - p0), E = n1 + 2 * Q;
  // halo mode (row slabs): Z^T holds the n1 + 2 Q extended rows (halo rows
  // from the neighbours / the global AR rows), column stride E
  const bool halo = a.halo != 0;
  const int zs = halo ? E : n1;
  const double* Z = reinterpret_cast<const double*>(a.zbuf) + (size_t)b * zs * n2;  // [c][row]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // stage interior rows rho in [rlo, rhi) at local l = rho + Q - p0 (cp.async, a column per warp pass)
  const int rlo = halo ? p0 - Q : max(0, p0 - Q), rhi = halo ? min(n1 + Q, p0 + NL - Q) : min(n1, p0 + NL - Q);
  const int lo = rlo + Q - p0, hi = rhi + Q - p0;
  for (int c = w; c < kColW; c += kColNT / 32) {
    if (c0 + c >= n2) break;
    const double* zc = Z + (size_t)(c0 + c) * zs + (halo ? Q : 0);
    for (int rho = rlo + lane; rho < rhi; rho += 32) cp_async8(smd + (rho + Q - p0) * kColLD + c, zc + rho);
  }
  cp_async_commit();
  cp_async_wait_all();
  __syncthreads();
  // extension rows (top band / bottom band) and zeros past the column or n2
  for (int idx = threadIdx.x; idx < (lo + NL - hi) * kColW; idx += kColNT) {
    const int e = idx / kColW, c = idx - e * kColW;
    const int l = e < lo ? e : hi + (e - lo), p = p0 + l, rho = p - Q;
    double v = 0.0;
    if (c0 + c < n2 && p < E && !halo) {
      if (a.bc == DBX_BC_REFLECTIVE) {
        v = smd[((rho < 0 ? -rho - 1 : 2 * n1 - 1 - rho) + Q - p0) * kColLD + c];
      } else {
        const int r0 = rho < 0 ? 0 : n1 - 1, ri = rho < 0 ? -rho : 2 * (n1 - 1) - rho;
        v = 2.0 * smd[(r0 + Q - p0) * kColLD + c] - smd[(ri + Q - p0) * kColLD + c];
      }
    }
    smd[l * kColLD + c] = v;
  }
  if (c0 + kColW > n2)
    for (int idx = threadIdx.x; idx < (hi - lo) * kColW; idx += kColNT) {
      const int l = lo + idx / kColW, c = idx % kColW;
      if (c0 + c >= n2) smd[l * kColLD + c] = 0.0;
    }
  __syncthreads();
  double* Y = (MODE == 0 ? reinterpret_cast<double*>(a.ybuf) + (size_t)b * N
                          : const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N))) +
              (size_t)p0 * n2 + c0 + lane;
  const double* G = MODE == 2 ? a.g + (size_t)b * N + (size_t)p0 * n2 + c0 + lane : nullptr;
  double p2 = 0.0;
  const bool colok = c0 + lane < n2;
  for (int i0 = w * RT; i0 < rows; i0 += (kColNT / 32) * RT) {
    const double* col = smd + i0 * kColLD + lane;
    double acc[RT];
#pragma unroll
    for (int r = 0; r < RT; ++r) acc[r] = 0.0;
#pragma unroll
    for (int s2 = 0; s2 < RT + 2 * Q; ++s2) {
      const double z = col[s2 * kColLD];
#pragma unroll
      for (int r = 0; r < RT; ++r) {
        const int t = s2 - r;
        if (t >= 0 && t < NTAP) acc[r] = fma(tp.t[t], z, acc[r]);
      }
    }
    if (colok) {
      if constexpr (MODE == 2) {
        // g loads four rows deep before their stores (the stores would keep
        // the compiler from hoisting them; 16 deep spills at 64 registers)
#pragma unroll
        for (int r0 = 0; r0 < RT; r0 += 4) {
          double gv[4];
#pragma unroll
          for (int r = 0; r < 4; ++r) gv[r] = i0 + r0 + r < rows ? __ldcs(G + (size_t)(i0 + r0 + r) * n2) : 0.0;
#pragma unroll
          for (int r = 0; r < 4; ++r)
            if (i0 + r0 + r < rows) {
              const double rv = gv[r] - acc[r0 + r];
              Y[(size_t)(i0 + r0 + r) * n2] = rv;
              p2 += rv * rv;
            }
        }
      } else {
#pragma unroll
        for (int r = 0; r < RT; ++r)
          if (i0 + r < rows) Y[(size_t)(i0 + r) * n2] = acc[r];
      }
    }
  }
  if constexpr (MODE == 2) {
    __shared__ double red[32];
    const double s2 = block_sum<kColNT>(p2, red);
    if (a.part.p && threadIdx.x == 0)
      a.part.p[(size_t)b * NUM_SLOTS * a.part.cap + SLOT_R2 * a.part.cap + blockIdx.z * gridDim.x + blockIdx.x] = s2;
  } else {
    (void)p2;
    (void)G;
  }
}

// Row pass of the separate-pass direct separable blur (any n2): FOUR rows x a
// segment of kRowSeg columns per CTA.  The segment and its 2 q2 halo columns
// are staged (halo columns past the image from the AR / reflective extension,
// boundary.hpp:56-64, read straight from global), then correlated with the
// row taps (sep_row_stencil_T) into Z^T ([c][row]) for cols_sep_real.
constexpr int kRowSeg = 1024, kRowNT = 256;
__host__ __device__ constexpr int rowseg_ls(int q2) {
  const int e = kRowSeg + 2 * q2 + 8;
  return e + ((4 - e % 16) + 16) % 16;  // stride = 4 mod 16 (sep_row_stencil_T bank pattern)
}

template <int Q>
__global__ void __launch_bounds__(kRowNT, 4) rows_sep_seg(SpecArgs a) {
  DBX_PDL_WAIT();
  const int b = blockIdx.z;
  if (a.st && a.st[b].done) return;
  extern __shared__ double smd[];
  const int n1 = a.n1, n2 = a.n2, LSX = rowseg_ls(Q);
  const int H = a.halo, ne = n1 + 2 * H;  // rows correlated (halo rows included)
  const size_t N = (size_t)n1 * n2;
  const int c0 = blockIdx.x * kRowSeg, r0 = blockIdx.y * 4;
  const int nl = min(4, ne - r0), nc = min(kRowSeg, n2 - c0), W = nc + 2 * Q;
  const double* X = resolve_ptr(a.in, a.st, a.insel, b, a.batch, N);
  // every global load of the CTA's staging in flight before the first
  // shared-memory store (one DRAM latency per thread instead of one per
  // element: the load -> store pairs of the rolled loop ran at 33 % of HBM)
  constexpr int NJ = (kRowSeg + 2 * Q + kRowNT - 1) / kRowNT;
  double v[4][NJ];
#pragma unroll
  for (int h = 0; h < 4; ++h) {
    const int re = r0 + h;  // extended row index: [0, H) top halo, [H, H + n1) slab, then bottom halo
    const double* xr = H == 0 ? X + (size_t)re * n2
                     : re < H ? a.htop + (size_t)re * n2
                     : re < H + n1 ? X + (size_t)(re - H) * n2 : a.hbot + (size_t)(re - H - n1) * n2;
#pragma unroll
    for (int i = 0; i < NJ; ++i) {
      const int j = threadIdx.x + i * kRowNT, c = c0 + j - Q;
      double x = 0.0;
      if (h < nl && j < W) {
        if (c >= 0 && c < n2) {
          x = __ldcs(xr + c);
        } else if (a.bc == DBX_BC_REFLECTIVE) {
          x = xr[c < 0 ? -c - 1 : 2 * n2 - 1 - c];
        } else {
          const int e = c < 0 ? 0 : n2 - 1, ri = c < 0 ? -c : 2 * (n2 - 1) - c;
          x = 2.0 * xr[e] - xr[ri];
        }
      }
      v[h][i] = x;
    }
  }
#pragma unroll
  for (int h = 0; h < 4; ++h)
#pragma unroll
    for (int i = 0; i < NJ; ++i) {
      const int j = threadIdx.x + i * kRowNT;
      if (j < W) smd[h * LSX + j] = v[h][i];
    }
  __syncthreads();
  sep_row_pass(smd, LSX, a.conv, Q, nc, nl, reinterpret_cast<double*>(a.zbuf) + (size_t)b * ne * n2 + (size_t)c0 * ne + r0,
               ne);
}

}  // namespace

// ---------------------------------------------------------------------------
// launchers (size dispatch)
// ---------------------------------------------------------------------------
#define DBX_CONV_LIST(X)                                                                       \
  X(64) X(72) X(80) X(96) X(128) X(144) X(160) X(192) X(256) X(270) X(288) X(320) X(384) X(512) \
  X(540) X(576) X(640) X(768) X(1024) X(1080) X(1152) X(1280) X(1536) X(2048) X(2160) X(2304) \
  X(2560) X(3072) X(4096) X(4320) X(4608) X(5120) X(6144) X(8192) X(8640)

int conv_supported_len(int need) {
  int best = 0;
#define X(L) if (best == 0 && (L) >= need) best = (L);
  DBX_CONV_LIST(X)
#undef X
  return best;
}

int launch_conv_row_fwd(const SpecArgs& a, cudaStream_t s) {
  const int L2 = a.conv.L2;
#define X(L)                                                                             \
  if (L2 == (L)) {                                                                       \
    constexpr int T = line_threads(L, 8), G = lines_for(L, kConvBudget, 8);                     \
    const size_t sm = ConvSmem<L, G>::row_bytes;                                         \
    static AttrOnce attr;                                                            \
    if (!attr.ensure(conv_row_fwd<L>, sm)) return -1;                            \
    dim3 grid((a.n1 + 2 * G - 1) / (2 * G), a.batch);                                    \
    launch_k(conv_row_fwd<L>, grid, T * G, sm, s, a);                                          \
    return (int)grid.x;                                                                  \
  }
  DBX_CONV_LIST(X)
#undef X
  return -1;
}

#define DBX_SEP_LIST(X) X(7) X(15)

bool conv_sep_supported(int q1) {
#define X(Q) if (q1 == (Q)) return true;
  DBX_SEP_LIST(X)
#undef X
  return false;
}

template <int Q, int BAND, int MODE>
int launch_cols_sep_real_t(const SpecArgs& a, cudaStream_t s) {
  ColTaps<2 * Q + 1> tp;
  if (!a.conv.sepa_host) return -1;
  for (int t = 0; t < 2 * Q + 1; ++t) tp.t[t] = a.conv.sepa_host[t];
  const size_t sm = (size_t)(BAND + 2 * Q) * kColLD * 8;
  if (!set_smem(cols_sep_real<Q, BAND, MODE>, sm)) return -1;
  dim3 grid((a.n2 + kColW - 1) / kColW, a.batch, (a.n1 + BAND - 1) / BAND);
  launch_k(cols_sep_real<Q, BAND, MODE>, grid, kColNT, sm, s, a, tp);
  return MODE == 2 ? (int)(grid.x * grid.z) : (int)grid.x;
}

// row band per CTA: 256 (2 CTAs / SM) or 128 (4 CTAs / SM); DBX_COL_BAND overrides
static int col_band() {
  static int band = [] {
    const char* e = getenv("DBX_COL_BAND");
    const int v = e ? atoi(e) : 128;
    return v == 256 ? 256 : 128;
  }();
  return band;
}

int launch_cols_sep_real(const SpecArgs& a, cudaStream_t s) {
#define X(Q)                                                                             \
  if (a.q1 == (Q))                                                                       \
    return col_band() == 256 ? launch_cols_sep_real_t<Q, 256, 0>(a, s) : launch_cols_sep_real_t<Q, 128, 0>(a, s);
  DBX_SEP_LIST(X)
#undef X
  return -1;
}

int launch_cols_sep_epi(const SpecArgs& a, int resid, cudaStream_t s) {
#define X(Q)                                                                             \
  if (a.q1 == (Q))                                                                       \
    return resid ? launch_cols_sep_real_t<Q, 128, 2>(a, s) : launch_cols_sep_real_t<Q, 128, 1>(a, s);
  DBX_SEP_LIST(X)
#undef X
  return -1;
}

bool rows_sep_supported(int q2) { return q2 == 7 || q2 == 15; }

int launch_rows_sep_seg(const SpecArgs& a, cudaStream_t s) {
  dim3 grid((a.n2 + kRowSeg - 1) / kRowSeg, (a.n1 + 2 * a.halo + 3) / 4, a.batch);
  const size_t sm = (size_t)4 * rowseg_ls(a.q2) * 8;
  if (a.q2 == 15) launch_k(rows_sep_seg<15>, grid, kRowNT, sm, s, a);
  else if (a.q2 == 7) launch_k(rows_sep_seg<7>, grid, kRowNT, sm, s, a);
  else return -1;
  return (int)(grid.x * grid.y);
}

int launch_conv_col(const SpecArgs& a, cudaStream_t s) {
  const int L1 = a.conv.L1;
  if (a.conv.sepa) {
    const int nb = sep_bands(a.n1);
    const size_t sm = (size_t)kSepCK * sep_stride(sep_band(a.n1, nb), a.q1) * 16;
#define X(Q)                                                                             \
    if (a.q1 == (Q)) {                                                                   \
      if (!set_smem(conv_col_sep<Q>, sm)) return -1;                                     \
      dim3 grid((a.conv.Lh + kSepCK - 1) / kSepCK, a.batch, nb);                         \
      launch_k(conv_col_sep<Q>, grid, kSepNT, sm, s, a);                                       \
      return (int)grid.x;                                                                \
    }
    DBX_SEP_LIST(X)
#undef X
    return -1;
  }
#define X(L)                                                                             \
  if (L1 == (L)) {                                                                       \
    constexpr int T = line_threads(L, 8), G = lines_for(L, kConvBudget, 8);                     \
    const size_t sm = ConvSmem<L, G>::col_bytes;                                         \
    static AttrOnce attr;                                                            \
    if (!attr.ensure(conv_col<L>, sm)) return -1;                                \
    dim3 grid((a.conv.Lh + G - 1) / G, a.batch);                                         \
    launch_k(conv_col<L>, grid, T * G, sm, s, a);                                              \
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
    static AttrOnce attr;                                                            \
    if (!attr.ensure(conv_row_inv<L>, sm)) return -1;                            \
    dim3 grid((a.n1 + 2 * G - 1) / (2 * G), a.batch);                                    \
    launch_k(conv_row_inv<L>, grid, T * G, sm, s, a);                                          \
    return (int)grid.x;                                                                  \
  }
  DBX_CONV_LIST(X)
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
