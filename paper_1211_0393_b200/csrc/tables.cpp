// tables.cpp — host-side precomputation for the FFT-form kernels (plan setup,
// not on the timed path).  All angles use exact integer argument reduction and
// long double evaluation, so every table entry is the correctly rounded double
// (naive sin(s t pi/(m+1)) arguments would burn ~1e-13 of the
// parity budget at the config lengths).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <thread>
#include <vector>

#include "tables.h"
#include "radix.h"

namespace dbx {
namespace {
constexpr long double kPiL = 3.141592653589793238462643383279502884L;

inline void put(double* out, long i, long double re, long double im) {
  out[2 * i] = (double)re;
  out[2 * i + 1] = (double)im;
}

template <typename F>
void parallel_for(long n, F f) {
  unsigned nt = std::thread::hardware_concurrency();
  if (nt == 0) nt = 1;
  if (nt > 32) nt = 32;
  if (n < 64 || nt == 1) {
    f(0, n);
    return;
  }
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) th.emplace_back(f, n * t / nt, n * (t + 1) / nt);
  for (auto& x : th) x.join();
}
}  // namespace

std::vector<double> twiddles(int L) {
  std::vector<double> tw(2 * (size_t)L);
  for (long e = 0; e < L; ++e) {
    const long double a = 2.0L * kPiL * (long double)e / (long double)L;
    put(tw.data(), e, cosl(a), -sinl(a));
  }
  return tw;
}

// H[k2][k1] = conj(sum_{t,u} w(t,u) exp(-2 pi i (k1 t / L1 + k2 u / L2))) / (L1 L2)
// (stored k2-major so a column pass reads its spectrum column contiguously)
std::vector<double> conv_spectrum(const double* w, int q1, int q2, int L1, int L2) {
  const int Lh = L2 / 2 + 1, H1 = 2 * q1 + 1, W2 = 2 * q2 + 1;
  std::vector<std::complex<long double>> e1((size_t)L1), e2((size_t)L2);
  for (long e = 0; e < L1; ++e) {
    const long double a = 2.0L * kPiL * (long double)e / (long double)L1;
    e1[(size_t)e] = {cosl(a), -sinl(a)};
  }
  for (long e = 0; e < L2; ++e) {
    const long double a = 2.0L * kPiL * (long double)e / (long double)L2;
    e2[(size_t)e] = {cosl(a), -sinl(a)};
  }
  // V(t, k2) = sum_u w(t,u) e2[k2 u]
  std::vector<std::complex<long double>> V((size_t)H1 * Lh);
  for (int t = 0; t < H1; ++t)
    for (int k2 = 0; k2 < Lh; ++k2) {
      std::complex<long double> acc = 0;
      for (int u = 0; u < W2; ++u) acc += (long double)w[t * W2 + u] * e2[(size_t)(((long)k2 * u) % L2)];
      V[(size_t)t * Lh + k2] = acc;
    }
  std::vector<double> H(2 * (size_t)L1 * Lh);
  const long double s = 1.0L / ((long double)L1 * (long double)L2);
  parallel_for(L1, [&](long b, long e) {
    for (long k1 = b; k1 < e; ++k1)
      for (int k2 = 0; k2 < Lh; ++k2) {
        std::complex<long double> acc = 0;
        for (int t = 0; t < H1; ++t) acc += e1[(size_t)((k1 * t) % L1)] * V[(size_t)t * Lh + k2];
        put(H.data(), (long)k2 * L1 + k1, acc.real() * s, -acc.imag() * s);  // [k2][k1]
      }
  });
  return H;
}

bool rank1_factor(const double* w, int q1, int q2, int L2, double tol, std::vector<double>& a,
                  std::vector<double>& beta, double* resid, std::vector<double>* brow) {
  const int H1 = 2 * q1 + 1, W2 = 2 * q2 + 1, Lh = L2 / 2 + 1;
  int i0 = 0, j0 = 0;
  double mx = 0.0;
  for (int t = 0; t < H1; ++t)
    for (int u = 0; u < W2; ++u)
      if (std::fabs(w[t * W2 + u]) > mx) mx = std::fabs(w[t * W2 + u]), i0 = t, j0 = u;
  if (mx == 0.0) return false;
  a.assign((size_t)H1, 0.0);
  std::vector<double> bf((size_t)W2);
  for (int t = 0; t < H1; ++t) a[(size_t)t] = w[t * W2 + j0];
  for (int u = 0; u < W2; ++u) bf[(size_t)u] = w[i0 * W2 + u] / w[i0 * W2 + j0];
  double r = 0.0;
  for (int t = 0; t < H1; ++t)
    for (int u = 0; u < W2; ++u) r = std::max(r, std::fabs(w[t * W2 + u] - a[(size_t)t] * bf[(size_t)u]));
  if (resid) *resid = r / mx;
  if (r > tol * mx) return false;
  if (brow) *brow = bf;
  beta.assign(2 * (size_t)Lh, 0.0);
  for (int k2 = 0; k2 < Lh; ++k2) {
    std::complex<long double> acc = 0;
    for (int u = 0; u < W2; ++u) {
      const long double ang = 2.0L * kPiL * (long double)(((long)k2 * u) % L2) / (long double)L2;
      acc += (long double)bf[(size_t)u] * std::complex<long double>(cosl(ang), -sinl(ang));
    }
    beta[2 * (size_t)k2] = (double)(acc.real() / (long double)L2);
    beta[2 * (size_t)k2 + 1] = (double)(-acc.imag() / (long double)L2);
  }
  return true;
}

void blue_chirp(BlueHost& b, long N, int M);
void ar_ramp(BlueHost& b, int n, bool sine_i);

// The kernel spectrum in the in-place Cooley-Tukey core's digit-reversed
// position order (radix.h ct_freq_of_pos; fft.cuh ct_convolve).
void ct_permute(BlueHost& b) {
  const int M = b.M;
  b.bct.assign(2 * (size_t)M, 0.0);
  for (int p = 0; p < M; ++p) {
    const int k = fft::ct_freq_of_pos(M, p);
    b.bct[2 * (size_t)p] = b.bhat[2 * (size_t)k];
    b.bct[2 * (size_t)p + 1] = b.bhat[2 * (size_t)k + 1];
  }
  // unpadded long lines (fft.cuh ct_nopad): the same spectrum element-major,
  // bctT[r][b] = bct[b R + r] with R the last level's radix, so the fused
  // product pass reads consecutive butterflies b from consecutive addresses
  if (fft::ct_nopad(M)) {
    int R = M;
    while (R / fft::ct_radix(R) > 1) R /= fft::ct_radix(R);
    const int NB = M / R;
    b.bctT.assign(2 * (size_t)M, 0.0);
    for (int blk = 0; blk < NB; ++blk)
      for (int r = 0; r < R; ++r) {
        const size_t src = (size_t)blk * R + r, dst = (size_t)r * NB + blk;
        b.bctT[2 * dst] = b.bct[2 * src];
        b.bctT[2 * dst + 1] = b.bct[2 * src + 1];
      }
  }
}

BlueHost bluestein(int n, bool sine_i, int M) {
  BlueHost b;
  b.n = n;
  b.N = sine_i ? n + 1 : n - 1;
  b.M = M;
  const long N = b.N;
  b.core = M == N ? 0 : 1;
  b.scale = (double)sqrtl(2.0L / (long double)N);
  b.tw = twiddles(M);
  if (M == N) {  // direct odd-length DFT: no chirp / kernel spectrum
    b.chirp.assign(2, 0.0);
    b.bhat.assign(2, 0.0);
    // level-1 twiddles of the warp-owned two-level DFTs, transposed (wdst.cu)
    const int n1n = N == 1023 ? 33 : N == 255 ? 15 : 0, n2n = N == 1023 ? 31 : 17;
    if (n1n) {
      // N = 1023: 15 more rows [j - 1][lane k2] = W_31^{j k2} for the 33rd level-2 row
      // N = 1023 also: rows 33..47 hold real weights (doubles, [j - 1][lane],
      // at double offset 2 * 32 * 48 + 32 (j - 1) + lane) of the split 33rd row:
      // lanes k2 <= 15 the cosines cos(2 pi j k2 / 31), lanes 16..30 the sines
      // sin(2 pi j (31 - lane) / 31) of their partner k2 = 31 - lane, lane 31 zero
      b.tw1t.assign(2 * 32 * (size_t)(n1n + (N == 1023 ? 15 : 0)) + (N == 1023 ? 15 * 32 : 0), 0.0);
      if (N == 1023)
        for (int j = 1; j <= 15; ++j) {
          for (int k2 = 0; k2 < 31; ++k2) {
            const size_t e = 33 * (size_t)((j * k2) % 31), o = (size_t)(33 + j - 1) * 32 + k2;
            b.tw1t[2 * o] = b.tw[2 * e];
            b.tw1t[2 * o + 1] = b.tw[2 * e + 1];
          }
          for (int lane = 0; lane < 31; ++lane) {
            const int k2 = lane <= 15 ? lane : 31 - lane;
            const size_t e = 33 * (size_t)((j * k2) % 31);  // tw[e] = (cos, -sin)(2 pi (j k2 mod 31) / 31)
            b.tw1t[2 * 32 * 48 + (size_t)(j - 1) * 32 + lane] = lane <= 15 ? b.tw[2 * e] : -b.tw[2 * e + 1];
          }
        }
      for (int k1 = 0; k1 < n1n; ++k1)
        for (int n2 = 0; n2 < n2n; ++n2) {
          const size_t e = (size_t)n2 * k1, o = (size_t)k1 * 32 + n2;
          b.tw1t[2 * o] = b.tw[2 * e];
          b.tw1t[2 * o + 1] = b.tw[2 * e + 1];
        }
    }
  } else {
    blue_chirp(b, N, M);
    ct_permute(b);
  }
  ar_ramp(b, n, sine_i);
  // sine pre-twiddle of the packed real DST (spectral_common.cuh, pk_fill)
  b.sn.assign((size_t)N, 0.0);
  for (long j = 1; j < N; ++j) b.sn[(size_t)j] = (double)sinl(kPiL * (long double)j / (long double)N);
  return b;
}

bool is_prime(long N) {
  if (N < 2) return false;
  for (long d = 2; d * d <= N; ++d)
    if (N % d == 0) return false;
  return true;
}

static long powmod(long a, long e, long m) {
  long r = 1 % m;
  a %= m;
  while (e > 0) {
    if (e & 1) r = (long)((__int128)r * a % m);
    a = (long)((__int128)a * a % m);
    e >>= 1;
  }
  return r;
}

BlueHost rader(int n, bool sine_i) {
  BlueHost b;
  b.n = n;
  b.N = sine_i ? n + 1 : n - 1;
  const long N = b.N, M = N - 1;
  b.M = (int)M;
  b.core = 2;
  b.scale = (double)sqrtl(2.0L / (long double)N);
  b.tw = twiddles((int)M);
  // primitive root: g^(M/q) != 1 for every prime factor q of M
  std::vector<long> qs;
  for (long m = M, d = 2; m > 1; ++d) {
    if (d * d > m) d = m;
    if (m % d == 0) {
      qs.push_back(d);
      while (m % d == 0) m /= d;
    }
  }
  long g = 2;
  for (;; ++g) {
    bool ok = true;
    for (long q : qs) ok = ok && powmod(g, M / q, N) != 1;
    if (ok) break;
  }
  b.dlog.assign((size_t)N, 0);
  b.ridx.assign((size_t)N, 0);
  std::vector<long> gp((size_t)M);  // g^p
  long v = 1;
  for (long p = 0; p < M; ++p) {
    gp[(size_t)p] = v;
    b.dlog[(size_t)v] = (int)p;
    v = v * g % N;
  }
  for (long l = 1; l < N; ++l) b.ridx[(size_t)l] = (int)((M - b.dlog[(size_t)l]) % M);
  // b_m = w^{g^-m}, g^-m = g^{(M - m) mod M}; bhat = FFT_M(b) / M
  std::vector<std::complex<long double>> bb((size_t)M), eM((size_t)M);
  for (long m = 0; m < M; ++m) {
    const long e = gp[(size_t)((M - m) % M)];
    const long double a = 2.0L * kPiL * (long double)e / (long double)N;
    bb[(size_t)m] = {cosl(a), -sinl(a)};
    const long double c = 2.0L * kPiL * (long double)m / (long double)M;
    eM[(size_t)m] = {cosl(c), -sinl(c)};
  }
  b.bhat.assign(2 * (size_t)M, 0.0);
  parallel_for(M, [&](long kb, long ke) {
    for (long k = kb; k < ke; ++k) {
      std::complex<long double> acc = 0;
      for (long t = 0; t < M; ++t) acc += bb[(size_t)t] * eM[(size_t)((k * t) % M)];
      acc /= (long double)M;
      put(b.bhat.data(), k, acc.real(), acc.imag());
    }
  });
  ct_permute(b);
  b.chirp.assign(2, 0.0);
  ar_ramp(b, n, sine_i);
  b.sn.assign((size_t)N, 0.0);
  for (long j = 1; j < N; ++j) b.sn[(size_t)j] = (double)sinl(kPiL * (long double)j / (long double)N);
  return b;
}

void blue_chirp(BlueHost& b, long N, int M) {
  b.chirp.assign(2 * (size_t)(N + 1), 0.0);
  std::vector<std::complex<long double>> w((size_t)N + 1);
  for (long j = 0; j <= N; ++j) {
    const long e = (j * j) % (2 * N);  // exact reduction of pi j^2 / N
    const long double a = kPiL * (long double)e / (long double)N;
    w[(size_t)j] = {cosl(a), -sinl(a)};
    put(b.chirp.data(), j, w[(size_t)j].real(), w[(size_t)j].imag());
  }
  // kernel c_t = conj(w_|t|) on t in (-N, N), wrapped mod M; bhat = FFT_M(c) / M
  std::vector<std::complex<long double>> c((size_t)M, 0);
  for (long t = 0; t < N; ++t) {
    c[(size_t)t] = std::conj(w[(size_t)t]);
    if (t) c[(size_t)(M - t)] = std::conj(w[(size_t)t]);
  }
  std::vector<std::complex<long double>> eM((size_t)M);
  for (long e = 0; e < M; ++e) {
    const long double a = 2.0L * kPiL * (long double)e / (long double)M;
    eM[(size_t)e] = {cosl(a), -sinl(a)};
  }
  b.bhat.assign(2 * (size_t)M, 0.0);
  parallel_for(M, [&](long kb, long ke) {
    for (long k = kb; k < ke; ++k) {
      std::complex<long double> acc = 0;
      for (long t = 0; t < M; ++t)
        if (c[(size_t)t] != std::complex<long double>(0)) acc += c[(size_t)t] * eM[(size_t)((k * t) % M)];
      acc /= (long double)M;
      put(b.bhat.data(), k, acc.real(), acc.imag());
    }
  });
}

// AR ramp (transforms.hpp:135-144), computed exactly as the reference does
void ar_ramp(BlueHost& b, int n, bool sine_i) {
  if (!sine_i) {
    b.p.assign((size_t)(n - 2), 0.0);
    double sq = 0.0;
    for (long j = 1; j <= n - 2; ++j) b.p[(size_t)(j - 1)] = 1.0 - (double)j / (double)(n - 1);
    for (double v : b.p) sq += v * v;
    b.alpha = std::sqrt(1.0 + sq);
  } else {
    b.p.assign(1, 0.0);
    b.alpha = 1.0;
  }
}


// Prime-factor (Good-Thomas) tables of the N-point DFT, N = N1 N2 coprime,
// N1 a compiled odd radix (row DFTs in registers), N2 prime with N2 - 1 a
// compiled in-place Cooley-Tukey length (column DFTs by Rader).  Line layout:
// N2 rows of N1 complex; row 0 holds n2 = 0, row 1 + p holds n2 = g^p (the
// Rader order), so the column convolutions read rows 1..N2-1 in place.
//   dlog[j] = row(n2) N1 + n1 with j = (N2 n1 + N1 n2) mod N (input map)
//   ridx[k2] = q with g^-q = k2 (mod N2), k2 in [1, N2): output U[k2] sits
//              at row 1 + q of its column (after the convolution)
//   tw      = W_{N2-1}^e, bct = FFT_{N2-1}(b) / (N2-1) in the CT core's
//             digit-reversed order, b_m = exp(-2 pi i g^-m / N2)
BlueHost pfa(int n, bool sine_i, int N1, int N2) {
  BlueHost b;
  b.n = n;
  b.N = sine_i ? n + 1 : n - 1;
  const long N = b.N, R = N2 - 1;
  b.M = (int)N;
  b.core = 3;
  b.scale = (double)sqrtl(2.0L / (long double)N);
  b.tw = twiddles((int)R);
  std::vector<long> qs;
  for (long m = R, d = 2; m > 1; ++d) {
    if (d * d > m) d = m;
    if (m % d == 0) {
      qs.push_back(d);
      while (m % d == 0) m /= d;
    }
  }
  long g = 2;
  for (;; ++g) {
    bool ok = true;
    for (long q : qs) ok = ok && powmod(g, R / q, N2) != 1;
    if (ok) break;
  }
  std::vector<long> dl((size_t)N2, 0), gp((size_t)R);
  long v = 1;
  for (long p = 0; p < R; ++p) {
    gp[(size_t)p] = v;
    dl[(size_t)v] = p;
    v = v * g % N2;
  }
  auto row = [&](long n2) { return n2 == 0 ? 0L : 1 + dl[(size_t)n2]; };
  // modular inverses by search (small moduli)
  long inv21 = 1, inv12 = 1;
  while ((N2 * inv21) % N1 != 1) ++inv21;
  while ((N1 * inv12) % N2 != 1) ++inv12;
  b.dlog.assign((size_t)N, 0);
  for (long j = 0; j < N; ++j) {
    const long n1 = (j % N1) * inv21 % N1, n2 = (j % N2) * inv12 % N2;
    b.dlog[(size_t)j] = (int)(row(n2) * N1 + n1);
  }
  b.ridx.assign((size_t)N2, 0);
  for (long k2 = 1; k2 < N2; ++k2) b.ridx[(size_t)k2] = (int)((R - dl[(size_t)k2]) % R);
  std::vector<std::complex<long double>> bb((size_t)R), eR((size_t)R);
  for (long m = 0; m < R; ++m) {
    const long e = gp[(size_t)((R - m) % R)];
    const long double a = 2.0L * kPiL * (long double)e / (long double)N2;
    bb[(size_t)m] = {cosl(a), -sinl(a)};
    const long double c = 2.0L * kPiL * (long double)m / (long double)R;
    eR[(size_t)m] = {cosl(c), -sinl(c)};
  }
  b.bhat.assign(2 * (size_t)R, 0.0);
  for (long k = 0; k < R; ++k) {
    std::complex<long double> acc = 0;
    for (long t = 0; t < R; ++t) acc += bb[(size_t)t] * eR[(size_t)((k * t) % R)];
    acc /= (long double)R;
    put(b.bhat.data(), k, acc.real(), acc.imag());
  }
  b.bct.assign(2 * (size_t)R, 0.0);
  for (int p = 0; p < (int)R; ++p) {
    const int k = fft::ct_freq_of_pos((int)R, p);
    b.bct[2 * (size_t)p] = b.bhat[2 * (size_t)k];
    b.bct[2 * (size_t)p + 1] = b.bhat[2 * (size_t)k + 1];
  }
  b.chirp.assign(2, 0.0);
  ar_ramp(b, n, sine_i);
  b.sn.assign((size_t)N, 0.0);
  for (long j = 1; j < N; ++j) b.sn[(size_t)j] = (double)sinl(kPiL * (long double)j / (long double)N);
  return b;
}

}  // namespace dbx
