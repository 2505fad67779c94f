// tables.h — host-side precomputation for the FFT-form kernels.
#pragma once

#include <vector>

namespace dbx {

// W_L^e = exp(-2 pi i e / L), e < L, interleaved (re, im).
std::vector<double> twiddles(int L);

// Kernel spectrum of the correlation weights w ((2q1+1) x (2q2+1), row-major):
// H[k2][k1] = conj(FFT2(w))[k1][k2] / (L1 L2), k1 < L1, k2 < L2/2 + 1 (k2-major).
std::vector<double> conv_spectrum(const double* w, int q1, int q2, int L1, int L2);
// Rank-1 factorisation w = a b^T of a (2 q1 + 1) x (2 q2 + 1) mask: true when
// max |w - a b^T| <= tol * max |w|.  a: column factor (2 q1 + 1); beta: the
// row factor's spectrum conj(B(k2)) / L2 for k2 < L2/2 + 1 (interleaved
// re/im), the per-column scale of the separable column pass; brow: the row
// factor b itself (2 q2 + 1) for a direct row pass.
bool rank1_factor(const double* w, int q1, int q2, int L2, double tol, std::vector<double>& a,
                  std::vector<double>& beta, double* resid, std::vector<double>* brow = nullptr);

struct BlueHost {
  int n = 0, N = 0, M = 0;
  double alpha = 1.0, scale = 1.0;
  std::vector<double> tw, chirp, bhat, p, sn;  // sn[j] = sin(pi j / N), j < N
  std::vector<double> bct;  // bhat in digit-reversed order (fft.cuh ct_convolve)
  std::vector<double> bctT; // bct element-major [r][block] for the unpadded long lines (tables.cpp ct_permute)
  // warp-owned DFT_1023 / DFT_255 (wdst.cu): level-1 twiddles W_N^{n2 k1} stored
  // [k1][32 lanes n2], so a warp's load of one k1 is one contiguous 512-byte row
  std::vector<double> tw1t;
  std::vector<int> dlog, ridx;                 // Rader permutations (prime N)
  int core = 0;                                // DstCore (spectral.h)
};

// Bluestein tables of the DST-I of one line: AR kinds (sine_i = false) use the
// interior of length n-2 (N = n-1); the plain SineI kind uses N = n+1.
BlueHost bluestein(int n, bool sine_i, int M);

// Rader tables of the same DST-I for prime N (M = N - 1): generator g of
// (Z/N)^*, dlog[j] = p with g^p = j, ridx[l] = q with g^-q = l, and the kernel
// spectrum bhat = FFT_M(b) / M, b_m = exp(-2 pi i g^-m / N).
BlueHost rader(int n, bool sine_i);
// Prime-factor tables (N = N1 N2, row DFTs of N1 in registers, column DFTs of
// the prime N2 by Rader over the in-place CT core): see tables.cpp pfa().
BlueHost pfa(int n, bool sine_i, int N1, int N2);
bool is_prime(long N);

}  // namespace dbx
