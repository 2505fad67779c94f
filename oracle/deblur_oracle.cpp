// ============================================================================
// oracle/deblur_oracle.cpp — CPU ORACLE (TEST INFRASTRUCTURE ONLY)
//
// This file is the parity checker for the B200 hot path.  It is a scalar,
// single-threaded C++ restatement of the reference library `deblur`
// (/root/reference/proj/include/deblur/*.hpp) for the anti-reflective (AR)
// preconditioned-Landweber path.  Only tests/, __graft_entry__.smoke() and the
// cpu_baseline / --impl reference legs of bench.py may load it; the product
// (paper_1211_0393_b200/libdbx.so) never links or calls it.
//
// The reference itself cannot be compiled here or on the GPU box (Eigen3,
// FFTW3 and GoogleTest are absent).  Its DST-I / DFT
// arithmetic lives in FFTW3 (unpinned, un-vendored: transforms.hpp:3, 39-82);
// this restatement computes the same unnormalised transforms with its own
// FFT (mixed radix + Bluestein), so results agree with FFTW to rounding.
// Parity pinning: the oracle is certified against the reference tests'
// known-answer and dense-formula assertions (tests/test_oracle_*.py) and
// against scipy.fft.dst(type=1) / committed golden fixtures at the BASELINE
// DST lengths (tests/golden/).
//
// Every function cites the reference file:line it restates.  Matrices are
// row-major double buffers (core.hpp:17-19: vec(X) is the buffer).
// ============================================================================
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstdint>
#include <cstring>
#include <limits>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using cd = std::complex<double>;
constexpr double kPi = 3.141592653589793238462643383279502884;  // core.hpp:15
constexpr long double kPiL = 3.141592653589793238462643383279502884L;

thread_local std::string g_err;

struct Mat {
  long n1 = 0, n2 = 0;
  std::vector<double> a;
  Mat() = default;
  Mat(long r, long c, double v = 0.0) : n1(r), n2(c), a(size_t(r * c), v) {}
  double& operator()(long i, long j) { return a[size_t(i * n2 + j)]; }
  double operator()(long i, long j) const { return a[size_t(i * n2 + j)]; }
};

// core.hpp:26-28
inline void require(bool c, const char* what) {
  if (!c) throw std::invalid_argument(what);
}

static double fro(const double* x, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += x[i] * x[i];
  return std::sqrt(s);
}

// ---------------------------------------------------------------------------
// Generic complex FFT (stands in for FFTW's fftw_plan_dft / r2r codelets,
// transforms.hpp:39-82).  Unnormalised, sign = -1 forward.
// ---------------------------------------------------------------------------
struct FftPlan {
  int n = 0, sign = -1;
  bool blue = false;
  std::vector<int> fac;
  std::vector<cd> tw;  // tw[k] = exp(sign*2*pi*i*k/n), k in [0,n)
  // Bluestein
  int M = 0;
  std::vector<cd> chirp;      // exp(sign*i*pi*k^2/n)
  std::vector<cd> kern_hat;   // FFT_M of conj chirp, wrapped
  std::shared_ptr<FftPlan> fM, iM;
};

static cd twiddle(long k, long n, int sign) {
  k %= n;
  if (k < 0) k += n;
  long double a = 2.0L * kPiL * (long double)k / (long double)n;
  return cd((double)cosl(a), (double)(sign * sinl(a)));
}

static std::shared_ptr<FftPlan> get_plan(int n, int sign);

static void fft_exec(const FftPlan& P, cd* x);

static std::shared_ptr<FftPlan> make_plan(int n, int sign) {
  auto P = std::make_shared<FftPlan>();
  P->n = n;
  P->sign = sign;
  int m = n;
  std::vector<int> f;
  for (int p : {4, 2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31}) {
    while (m % p == 0) {
      f.push_back(p);
      m /= p;
    }
  }
  if (m != 1) {
    // remaining large prime factor(s): Bluestein chirp-z over a power of two
    P->blue = true;
    int M = 1;
    while (M < 2 * n - 1) M <<= 1;
    P->M = M;
    P->chirp.resize(n);
    const long two_n = 2L * n;
    for (long k = 0; k < n; ++k) {
      long e = (k * k) % two_n;  // exact integer argument reduction
      long double a = kPiL * (long double)e / (long double)n;
      P->chirp[k] = cd((double)cosl(a), (double)(sign * sinl(a)));
    }
    P->fM = get_plan(M, -1);
    P->iM = get_plan(M, +1);
    P->kern_hat.assign(M, cd(0, 0));
    for (long k = 0; k < n; ++k) {
      P->kern_hat[k] = std::conj(P->chirp[k]);
      if (k) P->kern_hat[M - k] = std::conj(P->chirp[k]);
    }
    fft_exec(*P->fM, P->kern_hat.data());
    return P;
  }
  P->fac = f;
  P->tw.resize(n);
  for (int k = 0; k < n; ++k) P->tw[k] = twiddle(k, n, sign);
  return P;
}

static std::mutex g_plan_mu;
static std::map<std::pair<int, int>, std::shared_ptr<FftPlan>> g_plans;

static std::shared_ptr<FftPlan> get_plan(int n, int sign) {
  {
    std::lock_guard<std::mutex> lk(g_plan_mu);
    auto it = g_plans.find({n, sign});
    if (it != g_plans.end()) return it->second;
  }
  auto p = make_plan(n, sign);
  std::lock_guard<std::mutex> lk(g_plan_mu);
  g_plans[{n, sign}] = p;
  return p;
}

// decimation in time, out-of-place recursion over the factor list
static void fft_rec(const FftPlan& P, const cd* in, long s, cd* out, int n, int lvl,
                    std::vector<cd>& tmp) {
  if (n == 1) {
    out[0] = in[0];
    return;
  }
  const int p = P.fac[lvl];
  const int m = n / p;
  for (int r = 0; r < p; ++r) fft_rec(P, in + r * s, s * p, out + r * m, m, lvl + 1, tmp);
  const long step = P.n / n;  // W_n^e = tw[e*step]
  cd z[32];
  for (int k = 0; k < m; ++k) {
    for (int r = 0; r < p; ++r) z[r] = out[r * m + k] * P.tw[(size_t)((long)r * k * step % P.n)];
    for (int t = 0; t < p; ++t) {
      cd acc = z[0];
      for (int r = 1; r < p; ++r) acc += z[r] * P.tw[(size_t)(((long)r * t % p) * (P.n / p))];
      tmp[(size_t)(k + (long)m * t)] = acc;
    }
  }
  for (int i = 0; i < n; ++i) out[i] = tmp[i];
}

static void fft_exec(const FftPlan& P, cd* x) {
  const int n = P.n;
  if (n == 1) return;
  if (P.blue) {
    const int M = P.M;
    std::vector<cd> a(M, cd(0, 0));
    for (int k = 0; k < n; ++k) a[k] = x[k] * P.chirp[k];
    fft_exec(*P.fM, a.data());
    for (int k = 0; k < M; ++k) a[k] *= P.kern_hat[k];
    fft_exec(*P.iM, a.data());
    const double inv = 1.0 / M;
    for (int k = 0; k < n; ++k) x[k] = a[k] * inv * P.chirp[k];
    return;
  }
  std::vector<cd> in(x, x + n), tmp(n);
  fft_rec(P, in.data(), 1, x, n, 0, tmp);
}

static void fft(cd* x, int n, int sign) { fft_exec(*get_plan(n, sign), x); }

// 2D unnormalised DFT, rows then columns (transforms.hpp:66-82, 229-249)
static void dft2(std::vector<cd>& a, long L1, long L2, int sign) {
  for (long r = 0; r < L1; ++r) fft(&a[size_t(r * L2)], (int)L2, sign);
  std::vector<cd> col(L1);
  for (long c = 0; c < L2; ++c) {
    for (long r = 0; r < L1; ++r) col[r] = a[size_t(r * L2 + c)];
    fft(col.data(), (int)L1, sign);
    for (long r = 0; r < L1; ++r) a[size_t(r * L2 + c)] = col[r];
  }
}

// ---------------------------------------------------------------------------
// PSF (psf.hpp)
// ---------------------------------------------------------------------------
struct Psf {
  long q1, q2;
  Mat t;  // (2q1+1) x (2q2+1), centre (q1,q2)
  double tap(long i1, long i2) const { return t(q1 + i1, q2 + i2); }  // psf.hpp:32
};

// psf.hpp:15-25 (validation) — kMassTol = 1e-12 (psf.hpp:34)
static Psf make_psf(const double* taps, long q1, long q2) {
  require(q1 >= 0 && q2 >= 0, "Psf: taps must have odd dimensions");
  Psf p{q1, q2, Mat(2 * q1 + 1, 2 * q2 + 1)};
  double s = 0.0;
  for (size_t i = 0; i < p.t.a.size(); ++i) {
    p.t.a[i] = taps[i];
    require(std::isfinite(taps[i]), "Psf: taps must be finite");
    require(taps[i] >= 0.0, "Psf: taps must be nonnegative");
  }
  // Eigen's sum() is a pairwise/vectorised reduction; the 1e-12 tolerance
  // makes the summation order irrelevant for the accept/reject decision.
  for (double v : p.t.a) s += v;
  require(std::abs(s - 1.0) <= 1e-12, "Psf: taps must sum to 1 (within 1e-12)");
  return p;
}

// psf.hpp:55-66
static double max_asymmetry(const Psf& p) {
  double worst = 0.0;
  for (long i1 = -p.q1; i1 <= p.q1; ++i1)
    for (long i2 = -p.q2; i2 <= p.q2; ++i2)
      worst = std::max(worst, std::abs(p.tap(i1, i2) - p.tap(std::labs(i1), std::labs(i2))));
  return worst;
}

// psf.hpp:71-85
static Psf symmetrize(const Psf& p) {
  Psf s{p.q1, p.q2, Mat(2 * p.q1 + 1, 2 * p.q2 + 1)};
  for (long i1 = 0; i1 <= p.q1; ++i1)
    for (long i2 = 0; i2 <= p.q2; ++i2) {
      const double avg =
          (p.tap(-i1, -i2) + p.tap(-i1, i2) + p.tap(i1, -i2) + p.tap(i1, i2)) / 4.0;
      s.t(p.q1 + i1, p.q2 + i2) = avg;
      s.t(p.q1 - i1, p.q2 + i2) = avg;
      s.t(p.q1 + i1, p.q2 - i2) = avg;
      s.t(p.q1 - i1, p.q2 - i2) = avg;
    }
  return s;
}

// psf.hpp:88-91 (taps().reverse())
static Psf rotate180(const Psf& p) {
  Psf r = p;
  std::reverse(r.t.a.begin(), r.t.a.end());
  return r;
}

// psf.hpp:98-109 (accumulation order: h00, axis-1, axis-2, cross terms)
static double symbol_real(const Psf& p, double x1, double x2) {
  double acc = p.tap(0, 0);
  for (long s1 = 1; s1 <= p.q1; ++s1) acc += 2.0 * p.tap(s1, 0) * std::cos(s1 * x1);
  for (long s2 = 1; s2 <= p.q2; ++s2) acc += 2.0 * p.tap(0, s2) * std::cos(s2 * x2);
  for (long s1 = 1; s1 <= p.q1; ++s1)
    for (long s2 = 1; s2 <= p.q2; ++s2)
      acc += 4.0 * p.tap(s1, s2) * std::cos(s1 * x1) * std::cos(s2 * x2);
  return acc;
}

// ---------------------------------------------------------------------------
// Boundary (boundary.hpp) — AR branch only (the north star is AR-only)
// ---------------------------------------------------------------------------
// boundary.hpp:66-81 (AR branch)
static void check_support_ar(long n1, long n2, long q1, long q2) {
  require(n1 >= 1 && n2 >= 1, "pad: empty image");
  require((q1 == 0 || q1 <= n1 - 2) && (q2 == 0 || q2 <= n2 - 2),
          "anti-reflective support condition violated (q > n-2)");
}

enum Bc { kReflective = 2, kAntiReflective = 3 };  // BoundaryCondition order, boundary.hpp:9

// boundary.hpp:66-81 (Reflective branch)
static void check_support_refl(long n1, long n2, long q1, long q2) {
  require(n1 >= 1 && n2 >= 1, "pad: empty image");
  require(q1 <= n1 && q2 <= n2, "reflective support condition violated (q > n)");
}

// boundary.hpp:88-102 with extend_axis Reflective (49-55): f_{1-i} = f_i,
// f_{n+i} = f_{n+1-i}; rows first, then columns of the widened image.
static Mat pad_refl(const Mat& f, long q1, long q2) {
  const long n1 = f.n1, n2 = f.n2;
  check_support_refl(n1, n2, q1, q2);
  Mat out(n1 + 2 * q1, n2 + 2 * q2);
  for (long r = 0; r < n1; ++r)
    for (long c = 0; c < n2; ++c) out(q1 + r, q2 + c) = f(r, c);
  for (long r = 0; r < n1; ++r) {
    double* b = &out(q1 + r, 0);
    for (long i = 1; i <= q2; ++i) {
      b[q2 - i] = b[q2 + i - 1];
      b[q2 + n2 - 1 + i] = b[q2 + n2 - i];
    }
  }
  for (long c = 0; c < n2 + 2 * q2; ++c)
    for (long i = 1; i <= q1; ++i) {
      out(q1 - i, c) = out(q1 + i - 1, c);
      out(q1 + n1 - 1 + i, c) = out(q1 + n1 - i, c);
    }
  return out;
}

// boundary.hpp:88-102 with extend_axis AR (56-62): rows (axis 2) of the FOV
// first, then every column (axis 1) of the widened image.
static Mat pad_ar(const Mat& f, long q1, long q2) {
  const long n1 = f.n1, n2 = f.n2;
  check_support_ar(n1, n2, q1, q2);
  Mat out(n1 + 2 * q1, n2 + 2 * q2);
  for (long r = 0; r < n1; ++r)
    for (long c = 0; c < n2; ++c) out(q1 + r, q2 + c) = f(r, c);
  if (q2 > 0)
    for (long r = 0; r < n1; ++r) {
      double* b = &out(q1 + r, 0);
      for (long i = 1; i <= q2; ++i) {
        b[q2 - i] = 2.0 * b[q2] - b[q2 + i];
        b[q2 + n2 - 1 + i] = 2.0 * b[q2 + n2 - 1] - b[q2 + n2 - 1 - i];
      }
    }
  if (q1 > 0)
    for (long c = 0; c < n2 + 2 * q2; ++c) {
      auto b = [&](long i) -> double& { return out(i, c); };
      for (long i = 1; i <= q1; ++i) {
        b(q1 - i) = 2.0 * b(q1) - b(q1 + i);
        b(q1 + n1 - 1 + i) = 2.0 * b(q1 + n1 - 1) - b(q1 + n1 - 1 - i);
      }
    }
  return out;
}

// ---------------------------------------------------------------------------
// Blur (blur.hpp)
// ---------------------------------------------------------------------------
// blur.hpp:39-52
static Mat correlate_valid_direct(const Mat& P, const Psf& p, long n1, long n2) {
  const long q1 = p.q1, q2 = p.q2;
  Mat g(n1, n2);
  for (long r = 0; r < n1; ++r)
    for (long c = 0; c < n2; ++c) {
      double acc = 0.0;
      for (long s1 = -q1; s1 <= q1; ++s1)
        for (long s2 = -q2; s2 <= q2; ++s2) acc += p.tap(s1, s2) * P(r + q1 - s1, c + q2 - s2);
      g(r, c) = acc;
    }
  return g;
}

// blur.hpp:56-68: zero-embed in (rows+2q1) x (cols+2q2), DFT product, crop
static Mat correlate_valid_fft(const Mat& P, const Psf& p, long n1, long n2) {
  const long q1 = p.q1, q2 = p.q2;
  const long L1 = P.n1 + 2 * q1, L2 = P.n2 + 2 * q2;
  std::vector<cd> a(size_t(L1 * L2), cd(0, 0)), k(size_t(L1 * L2), cd(0, 0));
  for (long r = 0; r < P.n1; ++r)
    for (long c = 0; c < P.n2; ++c) a[size_t(r * L2 + c)] = P(r, c);
  for (long r = 0; r < 2 * q1 + 1; ++r)
    for (long c = 0; c < 2 * q2 + 1; ++c) k[size_t(r * L2 + c)] = p.t(r, c);
  dft2(a, L1, L2, -1);
  dft2(k, L1, L2, -1);
  for (size_t i = 0; i < a.size(); ++i) a[i] *= k[i];
  dft2(a, L1, L2, +1);
  const double inv = 1.0 / double(L1 * L2);
  Mat g(n1, n2);
  for (long r = 0; r < n1; ++r)
    for (long c = 0; c < n2; ++c) g(r, c) = (a[size_t((r + 2 * q1) * L2 + c + 2 * q2)] * inv).real();
  return g;
}

constexpr long kDirectConvMaxQ = 7;  // blur.hpp:70

// blur.hpp:75-83 (path: 0 auto, 1 direct, 2 fft)
static Mat apply(const Psf& p, const Mat& f, int path = 0, int bc = kAntiReflective) {
  const Mat P = bc == kReflective ? pad_refl(f, p.q1, p.q2) : pad_ar(f, p.q1, p.q2);
  const bool direct = path == 1 || (path == 0 && p.q1 <= kDirectConvMaxQ && p.q2 <= kDirectConvMaxQ);
  return direct ? correlate_valid_direct(P, p, f.n1, f.n2) : correlate_valid_fft(P, p, f.n1, f.n2);
}

// ---------------------------------------------------------------------------
// Transforms (transforms.hpp)
// ---------------------------------------------------------------------------
// FFTW RODFT00 semantics: y_k = 2 sum_j x_j sin(pi (j+1)(k+1)/(m+1)),
// computed through the 2(m+1)-point DFT of the odd extension.
static void rodft00(const double* x, double* y, long m) {
  const long N = m + 1, L = 2 * N;
  std::vector<cd> v(size_t(L), cd(0, 0));
  for (long j = 0; j < m; ++j) {
    v[size_t(j + 1)] = x[j];
    v[size_t(L - 1 - j)] = -x[j];
  }
  fft(v.data(), (int)L, -1);
  for (long k = 0; k < m; ++k) y[k] = -v[size_t(k + 1)].imag();
}

// transforms.hpp:114-121
static void sine1_forward(const double* v, double* y, long m) {
  require(m >= 1, "sine1_forward: empty input");
  rodft00(v, y, m);
  const double s = 0.5 * std::sqrt(2.0 / double(m + 1));
  for (long i = 0; i < m; ++i) y[i] *= s;
}

// transforms.hpp:129-144
struct ArT {
  long m = 0;
  double alpha = 1.0;
  std::vector<double> p;
};
static ArT make_ar_transform(long m) {
  require(m >= 3, "ArTransform1D: size must be at least 3");
  ArT t;
  t.m = m;
  t.p.resize(size_t(m - 2));
  double sq = 0.0;
  for (long j = 1; j <= m - 2; ++j) t.p[size_t(j - 1)] = 1.0 - double(j) / double(m - 1);
  for (double v : t.p) sq += v * v;  // Eigen squaredNorm: order differs only by rounding
  t.alpha = std::sqrt(1.0 + sq);
  return t;
}

// transforms.hpp:148-160
static void ar_forward(const ArT& t, const double* v, double* w) {
  const long m = t.m;
  const double inv_a = 1.0 / t.alpha;
  std::vector<double> in(v + 1, v + m - 1), out(size_t(m - 2));
  sine1_forward(in.data(), out.data(), m - 2);
  const double a0 = inv_a * v[0], a1 = inv_a * v[m - 1];
  for (long j = 0; j < m - 2; ++j) {
    double s = out[size_t(j)];
    s += a0 * t.p[size_t(j)];
    s += a1 * t.p[size_t(m - 3 - j)];
    out[size_t(j)] = s;
  }
  w[0] = inv_a * v[0];
  w[m - 1] = inv_a * v[m - 1];
  for (long j = 0; j < m - 2; ++j) w[j + 1] = out[size_t(j)];
}

// transforms.hpp:163-173
static void ar_inverse(const ArT& t, const double* v, double* u) {
  const long m = t.m;
  std::vector<double> in(size_t(m - 2)), out(size_t(m - 2));
  for (long j = 0; j < m - 2; ++j) {
    double s = v[j + 1] - v[0] * t.p[size_t(j)];
    s -= v[m - 1] * t.p[size_t(m - 3 - j)];
    in[size_t(j)] = s;
  }
  sine1_forward(in.data(), out.data(), m - 2);
  u[0] = t.alpha * v[0];
  u[m - 1] = t.alpha * v[m - 1];
  for (long j = 0; j < m - 2; ++j) u[j + 1] = out[size_t(j)];
}

enum Kind { kCosineIII = 1, kSineI = 2, kAR = 3, kARInv = 4 };  // TransformKind order, transforms.hpp:17

// transforms.hpp:88-110: R_m(s,t) = sqrt((2 - delta_{s,0})/m) cos(s (2t+1) pi / (2m))
// (0-based), FFTW REDFT10 / REDFT01 with the orthonormal scaling; restated
// as the dense definition with exact integer argument reduction (angle index
// s (2t+1) mod 4m) and long-double cosines.
static const std::vector<double>& cos4m(long m) {
  static thread_local std::map<long, std::vector<double>> cache;
  auto it = cache.find(m);
  if (it != cache.end()) return it->second;
  std::vector<double> c(size_t(4 * m));
  for (long e = 0; e < 4 * m; ++e) c[size_t(e)] = double(cosl(kPiL * (long double)e / (long double)(2 * m)));
  return cache.emplace(m, std::move(c)).first->second;
}
static void cosine3_forward(const double* v, double* y, long m) {
  require(m >= 1, "cosine3_forward: empty input");
  const auto& c = cos4m(m);
  const long double w0 = sqrtl(1.0L / (long double)m), w = sqrtl(2.0L / (long double)m);
  for (long s = 0; s < m; ++s) {
    long double acc = 0;
    for (long t = 0; t < m; ++t) acc += (long double)v[t] * c[size_t((s * (2 * t + 1)) % (4 * m))];
    y[s] = double(acc * (s == 0 ? w0 : w));
  }
}
static void cosine3_inverse(const double* v, double* y, long m) {
  require(m >= 1, "cosine3_inverse: empty input");
  const auto& c = cos4m(m);
  const long double w0 = sqrtl(1.0L / (long double)m), w = sqrtl(2.0L / (long double)m);
  for (long t = 0; t < m; ++t) {
    long double acc = (long double)v[0] * w0;
    for (long s = 1; s < m; ++s) acc += (long double)v[s] * w * c[size_t((s * (2 * t + 1)) % (4 * m))];
    y[t] = double(acc);
  }
}

// transforms.hpp:179-192 (columns first, then rows) + 198-226
static Mat tensor_apply(int kind, const Mat& x) {
  const long n1 = x.n1, n2 = x.n2;
  ArT t1, t2;
  if (kind == kAR || kind == kARInv) {
    require(n1 >= 3 && n2 >= 3, "tensor_apply: anti-reflective transform needs sizes >= 3");
    t1 = make_ar_transform(n1);
    t2 = make_ar_transform(n2);
  }
  auto kern = [&](const ArT& t, const double* in, double* out, long m) {
    if (kind == kCosineIII) cosine3_forward(in, out, m);
    else if (kind == -kCosineIII) cosine3_inverse(in, out, m);
    else if (kind == kSineI) sine1_forward(in, out, m);
    else if (kind == kAR) ar_forward(t, in, out);
    else ar_inverse(t, in, out);
  };
  Mat y(n1, n2);
  std::vector<double> buf(size_t(std::max(n1, n2))), o(size_t(std::max(n1, n2)));
  for (long c = 0; c < n2; ++c) {
    for (long r = 0; r < n1; ++r) buf[size_t(r)] = x(r, c);
    kern(t1, buf.data(), o.data(), n1);
    for (long r = 0; r < n1; ++r) y(r, c) = o[size_t(r)];
  }
  for (long r = 0; r < n1; ++r) {
    kern(t2, &y(r, 0), o.data(), n2);
    for (long c = 0; c < n2; ++c) y(r, c) = o[size_t(c)];
  }
  return y;
}

// ---------------------------------------------------------------------------
// Spectral / preconditioner (spectral.hpp, preconditioner.hpp)
// ---------------------------------------------------------------------------
// spectral.hpp:63-69
static std::vector<double> antireflective_grid(long m) {
  std::vector<double> x(size_t(m), 0.0);
  for (long r = 1; r <= m - 2; ++r) x[size_t(r)] = double(r) * kPi / double(m - 1);
  x[size_t(m - 1)] = 0.0;
  return x;
}

// spectral.hpp:120-133 + 43-48
static Mat eig_antireflective(const Psf& p, long n1, long n2) {
  require(max_asymmetry(p) <= 1e-12, "eig_antireflective: mask is not strongly symmetric");
  require(n1 >= 3 && n2 >= 3, "eig_antireflective: sizes must be >= 3");
  require(p.q1 <= n1 - 2 && p.q2 <= n2 - 2, "eig_antireflective: support condition violated");
  const auto x1 = antireflective_grid(n1), x2 = antireflective_grid(n2);
  Mat e(n1, n2);
  for (long a = 0; a < n1; ++a)
    for (long b = 0; b < n2; ++b) e(a, b) = symbol_real(p, x1[size_t(a)], x2[size_t(b)]);
  return e;
}

// spectral.hpp:50-54, 73-84: x_r = r pi / m, r = 0..m-1
static Mat eig_reflective(const Psf& p, long n1, long n2) {
  require(max_asymmetry(p) <= 1e-12, "eig_reflective: mask is not strongly symmetric");
  Mat e(n1, n2);
  for (long a = 0; a < n1; ++a)
    for (long b = 0; b < n2; ++b)
      e(a, b) = symbol_real(p, double(a) * kPi / double(n1), double(b) * kPi / double(n2));
  return e;
}

// preconditioner.hpp:37-57 (real algebra branch)
static Mat tikhonov_filter(const Mat& base, double alpha) {
  require(alpha >= 0.0, "tikhonov_filter: alpha must be nonnegative");
  bool allpos = true;
  for (double l : base.a) allpos = allpos && (l * l > 0.0);
  require(alpha > 0.0 || allpos, "tikhonov_filter: alpha = 0 with a zero eigenvalue");
  Mat d(base.n1, base.n2);
  for (size_t i = 0; i < d.a.size(); ++i) d.a[i] = 1.0 / (base.a[i] * base.a[i] + alpha);
  return d;
}

// preconditioner.hpp:62-85 (AntiReflective branch)
static Mat build_tikhonov(const Psf& p, double alpha, long n1, long n2) {
  const Psf s = symmetrize(p);
  return tikhonov_filter(eig_antireflective(s, n1, n2), alpha);
}

// preconditioner.hpp:62-85 (CosineIII branch)
static Mat build_tikhonov_cos(const Psf& p, double alpha, long n1, long n2) {
  const Psf s = symmetrize(p);
  return tikhonov_filter(eig_reflective(s, n1, n2), alpha);
}

// spectral.hpp:147-154: R^T diag(d) R (forward tensor, Hadamard, inverse tensor)
static Mat filter_apply_cos(const Mat& d, const Mat& x) {
  require(x.n1 == d.n1 && x.n2 == d.n2, "filter_apply: size mismatch");
  Mat xhat = tensor_apply(kCosineIII, x);
  for (size_t i = 0; i < xhat.a.size(); ++i) xhat.a[i] *= d.a[i];
  return tensor_apply(-kCosineIII, xhat);
}

// spectral.hpp:161-165 / preconditioner.hpp:88-90
static Mat filter_apply_ar(const Mat& d, const Mat& x) {
  require(x.n1 == d.n1 && x.n2 == d.n2, "filter_apply: size mismatch");
  Mat xhat = tensor_apply(kARInv, x);
  for (size_t i = 0; i < xhat.a.size(); ++i) xhat.a[i] *= d.a[i];
  return tensor_apply(kAR, xhat);
}

// ---------------------------------------------------------------------------
// Image model (image.hpp)
// ---------------------------------------------------------------------------
// image.hpp:44-66
struct GaussianSampler {
  std::mt19937_64 rng;
  double spare = 0.0;
  bool have = false;
  explicit GaussianSampler(uint64_t s) : rng(s) {}
  double operator()() {
    if (have) {
      have = false;
      return spare;
    }
    const double u1 = (double(rng() >> 11) + 1.0) * 0x1p-53;
    const double u2 = double(rng() >> 11) * 0x1p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * kPi * u2;
    spare = r * std::sin(a);
    have = true;
    return r * std::cos(a);
  }
};

// image.hpp:72-82
static void add_noise(const double* g, long n1, long n2, double level, uint64_t seed, double* out) {
  require(level >= 0.0, "add_noise: negative level");
  const size_t n = size_t(n1 * n2);
  if (level == 0.0) {
    std::memcpy(out, g, n * sizeof(double));
    return;
  }
  GaussianSampler gs(seed);
  std::vector<double> eta(n);
  for (size_t i = 0; i < n; ++i) eta[i] = gs();
  const double raw = fro(eta.data(), n);
  require(raw > 0.0, "add_noise: degenerate noise draw");
  const double s = level * fro(g, n) / raw;
  for (size_t i = 0; i < n; ++i) out[i] = g[i] + s * eta[i];
}

// image.hpp:85-91
static double rre(const double* x, const double* f, size_t n) {
  const double den = fro(f, n);
  require(den > 0.0, "rre: zero true image");
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += (x[i] - f[i]) * (x[i] - f[i]);
  return std::sqrt(s) / den;
}

}  // namespace orc

// ============================================================================
// extern "C" surface for ctypes (tests/, bench cpu_baseline only)
// Status: 0 ok, 1 invalid argument, 2 divergence.
// ============================================================================
using namespace orc;

#define ORC_TRY(...)                  \
  try {                               \
    __VA_ARGS__;                      \
    return 0;                         \
  } catch (const std::invalid_argument& e) { \
    g_err = e.what();                 \
    return 1;                         \
  } catch (const std::runtime_error& e) {    \
    g_err = e.what();                 \
    return 2;                         \
  }

static Mat to_mat(const double* x, long n1, long n2) {
  Mat m(n1, n2);
  std::memcpy(m.a.data(), x, sizeof(double) * size_t(n1 * n2));
  return m;
}
static void from_mat(const Mat& m, double* y) { std::memcpy(y, m.a.data(), sizeof(double) * m.a.size()); }

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_fft(double* re_im, int n, int sign) {
  ORC_TRY(fft(reinterpret_cast<cd*>(re_im), n, sign));
}

int orc_psf_check(const double* taps, int q1, int q2) { ORC_TRY(make_psf(taps, q1, q2)); }

int orc_symmetrize(const double* taps, int q1, int q2, double* out) {
  ORC_TRY(from_mat(symmetrize(make_psf(taps, q1, q2)).t, out));
}

int orc_pad_ar(const double* f, int n1, int n2, int q1, int q2, double* out) {
  ORC_TRY(from_mat(pad_ar(to_mat(f, n1, n2), q1, q2), out));
}

// path: 0 auto (reference cutover q<=7 direct), 1 direct, 2 fft
int orc_apply(const double* taps, int q1, int q2, const double* f, int n1, int n2, int adjoint,
              int path, double* out) {
  ORC_TRY({
    Psf p = make_psf(taps, q1, q2);
    require(n1 >= 1 && n2 >= 1, "BlurOperator: empty field of view");
    check_support_ar(n1, n2, q1, q2);
    if (adjoint) p = rotate180(p);
    from_mat(apply(p, to_mat(f, n1, n2), path), out);
  });
}

int orc_sine1(const double* v, int m, double* y) { ORC_TRY(sine1_forward(v, y, m)); }

int orc_ar_1d(int inverse, const double* v, int m, double* y) {
  ORC_TRY({
    ArT t = make_ar_transform(m);
    if (inverse) ar_inverse(t, v, y);
    else ar_forward(t, v, y);
  });
}

int orc_ar_alpha(int m, double* alpha, double* p) {
  ORC_TRY({
    ArT t = make_ar_transform(m);
    *alpha = t.alpha;
    if (p) std::memcpy(p, t.p.data(), sizeof(double) * t.p.size());
  });
}

int orc_tensor_apply(int kind, const double* x, int n1, int n2, double* y) {
  ORC_TRY({
    require(kind == kSineI || kind == kAR || kind == kARInv || kind == kCosineIII || kind == -kCosineIII,
            "tensor_apply: unsupported kind");
    from_mat(tensor_apply(kind, to_mat(x, n1, n2)), y);
  });
}

int orc_eig_antireflective(const double* taps, int q1, int q2, int n1, int n2, double* eigs) {
  ORC_TRY(from_mat(eig_antireflective(make_psf(taps, q1, q2), n1, n2), eigs));
}

int orc_tikhonov_filter(const double* eigs, int n1, int n2, double alpha, double* d) {
  ORC_TRY(from_mat(tikhonov_filter(to_mat(eigs, n1, n2), alpha), d));
}

int orc_build_tikhonov(const double* taps, int q1, int q2, int n1, int n2, double alpha, double* d) {
  ORC_TRY(from_mat(build_tikhonov(make_psf(taps, q1, q2), alpha, n1, n2), d));
}

int orc_precondition_apply(const double* d, const double* r, int n1, int n2, double* y) {
  ORC_TRY(from_mat(filter_apply_ar(to_mat(d, n1, n2), to_mat(r, n1, n2)), y));
}

int orc_add_noise(const double* g, int n1, int n2, double level, uint64_t seed, double* out) {
  ORC_TRY(add_noise(g, n1, n2, level, seed, out));
}

double orc_rre(const double* x, const double* f, long n) { return rre(x, f, size_t(n)); }

// solver.hpp:17-32 StoppingRule kinds
enum { STOP_FIXED = 0, STOP_MINRRE = 1, STOP_RESID = 2 };

// solver.hpp:63-132 landweber_loop (+ 139-148).  d == NULL -> plain
// Landweber.  x_hist (nullable) receives every iterate x_k, k = 1..executed.
// conv_path: 0 auto (reference cutover), 1 direct, 2 fft.
int orc_landweber_bc(const double* taps, int q1, int q2, int n1, int n2, const double* d,
                     const double* g, const double* f_true, double tau, int max_iters, int stop_kind,
                     int fixed_iters, double resid_eps, int conv_path, int bc, double* restored,
                     double* rre_hist, double* res_hist, int* best_iter, int* iters_done,
                     double* x_hist) {
  *iters_done = 0;
  *best_iter = 0;
  ORC_TRY({
    Psf p = make_psf(taps, q1, q2);
    require(n1 >= 1 && n2 >= 1, "BlurOperator: empty field of view");
    require(bc == kReflective || bc == kAntiReflective, "landweber: unsupported boundary condition");
    if (bc == kReflective) check_support_refl(n1, n2, q1, q2);
    else check_support_ar(n1, n2, q1, q2);
    require(tau > 0.0, "landweber: tau must be positive");
    require(max_iters >= 1, "landweber: max_iters must be at least 1");
    require(stop_kind != STOP_FIXED || fixed_iters >= 0, "StoppingRule: negative iteration count");
    require(stop_kind != STOP_RESID || resid_eps > 0.0, "StoppingRule: threshold must be positive");
    const size_t N = size_t(n1) * size_t(n2);
    const int total = stop_kind == STOP_FIXED ? fixed_iters : max_iters;
    const Mat G = to_mat(g, n1, n2);
    const double g_norm = fro(g, N);
    const double guard = 1e8 * g_norm;
    const Psf rot = rotate180(p);
    Mat D;
    if (d) D = to_mat(d, n1, n2);
    Mat x(n1, n2), best(n1, n2), r = G;
    double best_rre = std::numeric_limits<double>::infinity();
    for (int k = 1; k <= total; ++k) {
      Mat step = apply(rot, r, conv_path, bc);
      if (d) step = bc == kReflective ? filter_apply_cos(D, step) : filter_apply_ar(D, step);
      for (size_t i = 0; i < N; ++i) x.a[i] += tau * step.a[i];
      const Mat ax = apply(p, x, conv_path, bc);
      for (size_t i = 0; i < N; ++i) r.a[i] = G.a[i] - ax.a[i];
      if (fro(x.a.data(), N) > guard && g_norm > 0.0)
        throw std::runtime_error("landweber: iterate exceeded 1e8 * ||g||");
      const double rn = fro(r.a.data(), N);
      res_hist[k - 1] = rn;
      if (f_true) {
        const double e = rre(x.a.data(), f_true, N);
        rre_hist[k - 1] = e;
        if (e < best_rre) {
          best_rre = e;
          *best_iter = k;
          if (stop_kind == STOP_MINRRE) best = x;
        }
      }
      if (x_hist) std::memcpy(x_hist + size_t(k - 1) * N, x.a.data(), N * sizeof(double));
      *iters_done = k;
      if (stop_kind == STOP_RESID && g_norm > 0.0 && rn / g_norm < resid_eps) break;
    }
    const Mat& out = (stop_kind == STOP_MINRRE && f_true && *best_iter > 0) ? best : x;
    from_mat(out, restored);
  });
}

int orc_landweber(const double* taps, int q1, int q2, int n1, int n2, const double* d,
                  const double* g, const double* f_true, double tau, int max_iters, int stop_kind,
                  int fixed_iters, double resid_eps, int conv_path, double* restored,
                  double* rre_hist, double* res_hist, int* best_iter, int* iters_done,
                  double* x_hist) {
  return orc_landweber_bc(taps, q1, q2, n1, n2, d, g, f_true, tau, max_iters, stop_kind, fixed_iters, resid_eps,
                          conv_path, kAntiReflective, restored, rre_hist, res_hist, best_iter, iters_done, x_hist);
}

// Reflective BC / CosineIII algebra (the paper's comparison path)
int orc_apply_bc(const double* taps, int q1, int q2, const double* f, int n1, int n2, int adjoint, int path,
                 int bc, double* out) {
  ORC_TRY({
    require(bc == kReflective || bc == kAntiReflective, "apply: unsupported boundary condition");
    Psf p = make_psf(taps, q1, q2);
    if (adjoint) p = rotate180(p);
    from_mat(apply(p, to_mat(f, n1, n2), path, bc), out);
  });
}

int orc_build_tikhonov_bc(const double* taps, int q1, int q2, int n1, int n2, double alpha, int bc, double* d) {
  ORC_TRY({
    require(bc == kReflective || bc == kAntiReflective, "build_tikhonov: unsupported boundary condition");
    const Psf p = make_psf(taps, q1, q2);
    from_mat(bc == kReflective ? build_tikhonov_cos(p, alpha, n1, n2) : build_tikhonov(p, alpha, n1, n2), d);
  });
}

int orc_precondition_apply_bc(const double* d, const double* r, int n1, int n2, int bc, double* y) {
  ORC_TRY({
    const Mat D = to_mat(d, n1, n2), R = to_mat(r, n1, n2);
    from_mat(bc == kReflective ? filter_apply_cos(D, R) : filter_apply_ar(D, R), y);
  });
}

int orc_cosine3(int inverse, const double* v, int m, double* y) {
  ORC_TRY(inverse ? cosine3_inverse(v, y, m) : cosine3_forward(v, y, m));
}

}  // extern "C"
