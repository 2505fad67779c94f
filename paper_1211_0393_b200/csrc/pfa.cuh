// pfa.cuh — prime-factor (Good-Thomas) N-point DFT core of the packed
// DST-I for N = N1 N2 with N1 a compiled odd radix and N2 a prime whose
// N2 - 1 is a compiled in-place Cooley-Tukey length: C4's 2047 = 23 x 89 and
// C2's 511 = 7 x 73 (instead of Bluestein over 4096 / 1024 points).
//
// Line layout (tables.cpp pfa()): N2 rows of N1 complex; row 0 holds n2 = 0,
// row 1 + p holds n2 = g^p (Rader order of the column index).  The packed
// fill scatters z_j to its (row, column) through dlog; then
//   rows:    N2 DFT-N1 in registers (dft_odd_store), outputs in place;
//   columns: N1 cyclic convolutions of length R = N2 - 1 (the Rader
//            sequences at rows 1..R, stride N1) on the in-place CT core
//            (forward DIF, kernel spectrum in digit-reversed order, DIT
//            inverse), threads mapped column-fastest;
//   row 0:   U[0] = u0 + sum of the Rader sequence (the DC of its forward FFT);
//            the other outputs lack u0, which pfa_get adds (u0 kept per line).
// Replaces (reference): the FFTW RODFT00 plans of sine1_forward
// (transforms.hpp:112-121, 28-53) for these lengths.
#pragma once

#include <cuda_runtime.h>

#include "fft.cuh"
#include "spectral.h"

namespace dbx {

// compiled prime-factor lengths (dst.cu DBX_PFA_LIST, fused.cu DBX_FUSED_LIST)
__host__ __device__ constexpr bool pfa_len(int M) { return M == 115 || M == 511 || M == 2047; }

template <int M>
struct Pfa {
  static constexpr int N1 = pfa_len(M) ? fft::next_radix(M) : 1;
  static constexpr int N2 = M / N1;
  static constexpr int R = N2 - 1;
};

// twiddle entries a DST core of line length M reads (the PFA columns read
// W_R^e of the CT core; the other cores their FFT's prefix)
__host__ __device__ constexpr int dst_twiddles_needed(int M) {
  return pfa_len(M) ? fft::ct_twiddles_needed(M / fft::next_radix(M) - 1) : fft::twiddles_needed(M);
}

template <int L, int Ls, int P, int T, int DIR>
__device__ __forceinline__ void ctm_level(double2* buf, const double2* __restrict__ tw, int t, int bar) {
  constexpr int R = fft::ct_radix(Ls), m = Ls / R, NB = L / R;
#pragma unroll 1
  for (int beta = t; beta < P * NB; beta += T) {
    const int bb = beta / P, prob = beta - bb * P;
    const int blk = bb / m, j = bb - blk * m;
    const int base = blk * Ls + j;
    const double2 w1 = tw[j * (L / Ls)];
    double2 v[R];
#pragma unroll
    for (int r = 0; r < R; ++r) v[r] = buf[(1 + base + r * m) * P + prob];
    if constexpr (DIR < 0) {
      fft::dft<R, -1>(v);
      fft::apply_twiddles<R, -1>(v, w1);
    } else {
      fft::apply_twiddles<R, +1>(v, w1);
      fft::dft<R, +1>(v);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) buf[(1 + base + r * m) * P + prob] = v[r];
  }
  fft::line_sync(bar, T);
}
template <int L, int Ls, int P, int T>
__device__ __forceinline__ void ctm_dif(double2* buf, const double2* __restrict__ tw, int t, int bar) {
  if constexpr (Ls / fft::ct_radix(Ls) > 1) {
    ctm_level<L, Ls, P, T, -1>(buf, tw, t, bar);
    ctm_dif<L, Ls / fft::ct_radix(Ls), P, T>(buf, tw, t, bar);
  }
}
template <int L, int Ls, int P, int T>
__device__ __forceinline__ void ctm_dit(double2* buf, const double2* __restrict__ tw, int t, int bar) {
  if constexpr (Ls / fft::ct_radix(Ls) > 1) {
    ctm_dit<L, Ls / fft::ct_radix(Ls), P, T>(buf, tw, t, bar);
    ctm_level<L, Ls, P, T, +1>(buf, tw, t, bar);
  }
}

// The N-point DFT of one PFA line by its T threads (t = thread in line; bar
// as fft::fft: 0 = whole CTA, > 0 = named barrier of the line).  aux: 2 N1
// double2 of shared memory per line (u0, then the columns' Rader sums); u0
// stays there for pfa_get.
template <int M, int T>
__device__ __forceinline__ void pfa_core(double2* buf, const BlueTables& bt, const double2* tw, int t, int bar,
                                         double2* aux) {
  using P = Pfa<M>;
  constexpr int N1 = P::N1, N2 = P::N2, R = P::R;
  double2* u0s = aux;
  double2* dcs = aux + N1;
#pragma unroll 1
  for (int r = t; r < N2; r += T) {
    double2 v[N1];
#pragma unroll
    for (int n1 = 0; n1 < N1; ++n1) v[n1] = buf[r * N1 + n1];
    fft::dft_odd_store<N1, -1, M>(v, buf, r * N1, 1);
  }
  fft::line_sync(bar, T);
  if (t < N1) u0s[t] = buf[t];
  ctm_dif<R, R, N1, T>(buf, tw, t, bar);
  {
    constexpr int RL = fft::ct_last_radix<R>(), NB = R / RL;
#pragma unroll 1
    for (int beta = t; beta < N1 * NB; beta += T) {
      const int bb = beta / N1, prob = beta - bb * N1;
      const int base = bb * RL;
      double2 v[RL];
#pragma unroll
      for (int r = 0; r < RL; ++r) v[r] = buf[(1 + base + r) * N1 + prob];
      fft::dft<RL, -1>(v);
      if (base == 0) dcs[prob] = v[0];  // sum of the column's Rader sequence
#pragma unroll
      for (int r = 0; r < RL; ++r) v[r] = fft::cmul(v[r], __ldg(bt.bct + base + r));
      fft::dft<RL, +1>(v);
#pragma unroll
      for (int r = 0; r < RL; ++r) buf[(1 + base + r) * N1 + prob] = v[r];
    }
    fft::line_sync(bar, T);
  }
  ctm_dit<R, R, N1, T>(buf, tw, t, bar);
  if (t < N1) buf[t] = fft::cadd(u0s[t], dcs[t]);
  fft::line_sync(bar, T);
}

// Z_l of a PFA line after pfa_core: k1 = l mod N1, k2 = l mod N2; row 0
// holds k2 = 0, row 1 + q holds k2 = g^-q without the column's u0.
template <int M>
__device__ __forceinline__ double2 pfa_get(const double2* buf, const BlueTables& bt, int l, const double2* u0) {
  using P = Pfa<M>;
  const int k1 = l % P::N1, k2 = l % P::N2;
  if (k2 == 0) return buf[k1];
  return fft::cadd(buf[(1 + __ldg(bt.ridx + k2)) * P::N1 + k1], u0[k1]);
}

}  // namespace dbx
