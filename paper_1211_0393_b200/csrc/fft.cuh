// fft.cuh — batched FP64 complex FFT of compile-time length L in shared memory.
//
// Stockham autosort, mixed radix {8, 4, 2, 3, 5}: every stage loads the
// thread's butterflies into registers, synchronises, applies the stage
// twiddles W_{Ns R}^{r k} (from a forward twiddle table W_L^e, e < L, built on
// the host in long double with exact integer argument reduction), runs the
// radix-R DFT in registers and stores in place.  Each line owns a padded smem
// buffer (index i -> i + i/8) so that the stride-R stores of the first stage
// do not serialise on one bank group.  T threads cooperate on one line; a CTA
// runs several lines in lock-step (every thread calls every stage, so the
// __syncthreads() inside are CTA-uniform).
//
// This engine stands in for FFTW (reference transforms.hpp:39-82, blur.hpp:56-68):
// it carries the FFT-correlation blur and the Bluestein DST-I of the AR
// transform on the GPU.
#pragma once

#include <cuda_runtime.h>

#include <type_traits>

#include "dft_consts.h"
#include "radix.h"

namespace dbx {

// Phase timing (instrumented builds only: -DDBX_PHASES): thread 0 of every CTA
// adds the clock64() delta since its previous mark to g_phase[i] (one
// namespace-scope shared timestamp per CTA, so marks may sit in any device
// function, e.g. after every FFT stage).
#ifdef DBX_PHASES
static __device__ unsigned long long g_phase[64];  // per translation unit (fused.cu reads its own)
static __shared__ unsigned long long ph_t0s;
#define PH_DECL \
  if (threadIdx.x == 0) ph_t0s = clock64();
#define PH(i)                                        \
  if (threadIdx.x == 0) {                            \
    const unsigned long long ph_t1 = clock64();      \
    atomicAdd(&g_phase[i], ph_t1 - ph_t0s);          \
    ph_t0s = ph_t1;                                  \
  }
#else
#define PH_DECL
#define PH(i)
#endif

namespace fft {

// Even lengths (power-of-two radices) pad one element per 8 so stride-8
// accesses spread over the banks; odd lengths (odd strides) are conflict-free
// unpadded, which keeps a butterfly's addresses base + immediate.
// L = 8190 (C5's Rader convolution, in-place CT core 13.7.15.3.2) stays
// unpadded: its two long levels walk unit-stride runs whose quarter-warp
// alignment the padding breaks (2-way conflicts), and the short levels are made
// conflict-free by the butterfly-to-lane maps in ct_level / ct_convolve instead
// (-DDBX_CT_NOPAD=0 restores the padded layout for the A/B).
// (ct_nopad lives in radix.h: the host tables need it too)
template <int L>
__host__ __device__ constexpr int pad(int i) { return ((L & 1) || ct_nopad(L)) ? i : i + (i >> 3); }
__host__ __device__ constexpr int padded_len(int L) { return (L & 1) ? L + 1 : L + (L >> 3) + 1; }

// threads per line: one radix-8 butterfly per thread, rounded to a warp
__host__ __device__ constexpr int threads_for(int L) {
  int t = (L / 8 + 31) / 32 * 32;
  return t < 32 ? 32 : (t > 512 ? 512 : t);
}

// Twiddle entries an FFT of length L reads: stage (Ns, R) reads W_L^{k L/(Ns R)},
// k < Ns (largest index (Ns-1) L/(Ns R)) — only that prefix of the table
// needs staging.
__host__ __device__ constexpr int twiddles_needed(int L) {
  int rem = L, Ns = 1, mx = 0;
  while (rem > 1) {
    const int r = next_radix(rem);
    if (r == 0) return L;
    const int top = (Ns - 1) * (L / (Ns * r));
    mx = top > mx ? top : mx;
    Ns *= r;
    rem /= r;
  }
  return mx + 1;
}

__host__ __device__ constexpr bool supported(int L) {
  if (L < 2) return false;
  while (L > 1) {
    const int r = next_radix(L);
    if (r == 0) return false;
    L /= r;
  }
  return true;
}

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// a * conj(b)
__device__ __forceinline__ double2 cmulc(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, a.y * b.y), fma(a.y, b.x, -a.x * b.y));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
// v * (S*i)
template <int S>
__device__ __forceinline__ double2 mul_si(double2 v) {
  return S < 0 ? make_double2(v.y, -v.x) : make_double2(-v.y, v.x);
}

template <int S>
__device__ __forceinline__ void dft2(double2* v) {
  const double2 a = v[0];
  v[0] = cadd(a, v[1]);
  v[1] = csub(a, v[1]);
}

template <int S>
__device__ __forceinline__ void dft4(double2& x0, double2& x1, double2& x2, double2& x3) {
  const double2 t0 = cadd(x0, x2), t1 = csub(x0, x2), t2 = cadd(x1, x3);
  const double2 t3 = mul_si<S>(csub(x1, x3));
  x0 = cadd(t0, t2);
  x2 = csub(t0, t2);
  x1 = cadd(t1, t3);
  x3 = csub(t1, t3);
}

template <int S>
__device__ __forceinline__ void dft8(double2* v) {
  constexpr double h = 0.70710678118654752440084436210484904;
  double2 e0 = v[0], e1 = v[2], e2 = v[4], e3 = v[6];
  double2 o0 = v[1], o1 = v[3], o2 = v[5], o3 = v[7];
  dft4<S>(e0, e1, e2, e3);
  dft4<S>(o0, o1, o2, o3);
  // W8^1 = h(1 + S i), W8^2 = S i, W8^3 = h(-1 + S i)
  const double2 w1 = make_double2(h * (o1.x - S * o1.y), h * (o1.y + S * o1.x));
  const double2 w2 = mul_si<S>(o2);
  const double2 w3 = make_double2(h * (-o3.x - S * o3.y), h * (-o3.y + S * o3.x));
  v[0] = cadd(e0, o0);
  v[4] = csub(e0, o0);
  v[1] = cadd(e1, w1);
  v[5] = csub(e1, w1);
  v[2] = cadd(e2, w2);
  v[6] = csub(e2, w2);
  v[3] = cadd(e3, w3);
  v[7] = csub(e3, w3);
}

template <int S>
__device__ __forceinline__ void dft3(double2* v) {
  constexpr double c = 0.86602540378443864676372317075293618;  // sqrt(3)/2
  const double2 t = cadd(v[1], v[2]);
  const double2 u = mul_si<S>(cscale(csub(v[1], v[2]), c));
  const double2 m = make_double2(v[0].x - 0.5 * t.x, v[0].y - 0.5 * t.y);
  v[0] = cadd(v[0], t);
  v[1] = cadd(m, u);
  v[2] = csub(m, u);
}

template <int S>
__device__ __forceinline__ void dft5(double2* v) {
  constexpr double c1 = 0.30901699437494742410229341718281906;    // cos(2pi/5)
  constexpr double c2 = -0.80901699437494742410229341718281906;   // cos(4pi/5)
  constexpr double s1 = 0.95105651629515357211643933337938214;    // sin(2pi/5)
  constexpr double s2 = 0.58778525229247312916870595463907277;    // sin(4pi/5)
  const double2 a1 = cadd(v[1], v[4]), b1 = csub(v[1], v[4]);
  const double2 a2 = cadd(v[2], v[3]), b2 = csub(v[2], v[3]);
  const double2 x0 = v[0];
  const double2 m1 = make_double2(x0.x + c1 * a1.x + c2 * a2.x, x0.y + c1 * a1.y + c2 * a2.y);
  const double2 m2 = make_double2(x0.x + c2 * a1.x + c1 * a2.x, x0.y + c2 * a1.y + c1 * a2.y);
  const double2 n1 = mul_si<S>(make_double2(s1 * b1.x + s2 * b2.x, s1 * b1.y + s2 * b2.y));
  const double2 n2 = mul_si<S>(make_double2(s2 * b1.x - s1 * b2.x, s2 * b1.y - s1 * b2.y));
  v[0] = cadd(x0, cadd(a1, a2));
  v[1] = cadd(m1, n1);
  v[4] = csub(m1, n1);
  v[2] = cadd(m2, n2);
  v[3] = csub(m2, n2);
}

// Radix 9 = 3 x 3 (Cooley-Tukey): DFT-3 over n1 for each n2, internal twiddles
// W9^{n2 k1}, DFT-3 over n2; output k = k1 + 3 k2 (natural order).
template <int S>
__device__ __forceinline__ void dft9(double2* v) {
  constexpr double c1 = 0.76604444311897803520239265055541667;   // cos(2pi/9)
  constexpr double s1 = 0.64278760968653932632264340990726343;   // sin(2pi/9)
  constexpr double c2 = 0.17364817766693034885171662676931480;   // cos(4pi/9)
  constexpr double s2 = 0.98480775301220805936674302458952301;   // sin(4pi/9)
  constexpr double c4 = -0.93969262078590838405410927732473147;  // cos(8pi/9)
  constexpr double s4 = 0.34202014332566873304409961468225958;   // sin(8pi/9)
  double2 y[3][3];
#pragma unroll
  for (int n2 = 0; n2 < 3; ++n2) {
    double2 t[3] = {v[n2], v[n2 + 3], v[n2 + 6]};
    dft3<S>(t);
    y[n2][0] = t[0];
    y[n2][1] = t[1];
    y[n2][2] = t[2];
  }
  y[1][1] = cmul(y[1][1], make_double2(c1, S * s1));
  y[1][2] = cmul(y[1][2], make_double2(c2, S * s2));
  y[2][1] = cmul(y[2][1], make_double2(c2, S * s2));
  y[2][2] = cmul(y[2][2], make_double2(c4, S * s4));
#pragma unroll
  for (int k1 = 0; k1 < 3; ++k1) {
    double2 t[3] = {y[0][k1], y[1][k1], y[2][k1]};
    dft3<S>(t);
    v[k1] = t[0];
    v[k1 + 3] = t[1];
    v[k1 + 6] = t[2];
  }
}

// Radix 6 = 2 x 3 prime-factor (no internal twiddles): input n = (3 n1 + 2 n2)
// mod 6, output k = (3 k1 + 4 k2) mod 6.  The last level of the in-place CT
// core when the chain ends in 6 (8190 = 13.7.15.6: one level, one barrier and
// two line passes fewer than 13.7.15.3.2).
template <int S>
__device__ __forceinline__ void dft6(double2* v) {
  double2 a[3] = {v[0], v[2], v[4]}, b[3] = {v[3], v[5], v[1]};
  dft3<S>(a);
  dft3<S>(b);
#pragma unroll
  for (int k2 = 0; k2 < 3; ++k2) {
    v[(4 * k2) % 6] = cadd(a[k2], b[k2]);
    v[(3 + 4 * k2) % 6] = csub(a[k2], b[k2]);
  }
}

// Radix 15 = 3 x 5 prime-factor (Good-Thomas, no internal twiddles): input
// n = (5 n1 + 3 n2) mod 15, output k = (10 k1 + 6 k2) mod 15.
template <int S>
__device__ __forceinline__ void dft15(double2* v) {
  double2 y[5][3];
#pragma unroll
  for (int n2 = 0; n2 < 5; ++n2) {
    double2 t[3] = {v[(3 * n2) % 15], v[(5 + 3 * n2) % 15], v[(10 + 3 * n2) % 15]};
    dft3<S>(t);
    y[n2][0] = t[0];
    y[n2][1] = t[1];
    y[n2][2] = t[2];
  }
#pragma unroll
  for (int k1 = 0; k1 < 3; ++k1) {
    double2 u[5] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1], y[4][k1]};
    dft5<S>(u);
#pragma unroll
    for (int k2 = 0; k2 < 5; ++k2) v[(10 * k1 + 6 * k2) % 15] = u[k2];
  }
}

// Odd prime P >= 7 via the (P-1)/2 symmetric pairs:
//   X_k = x0 + sum_j c_jk a_j + S i sum_j s_jk b_j,  X_{P-k} = same with -S i,
//   a_j = x_j + x_{P-j}, b_j = x_j - x_{P-j}; ~2P real FMAs per element instead
//   of 4P for the plain matrix form.  Constants are compile-time (dft_consts.h).
template <int P, int S>
__device__ __forceinline__ void dft_odd(double2* v) {
  constexpr int H = (P - 1) / 2;
  using K = OddConst<P>;
  double2 a[H], b[H];
  const double2 x0 = v[0];
  double2 sum = x0;
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    a[j - 1] = cadd(v[j], v[P - j]);
    b[j - 1] = csub(v[j], v[P - j]);
    sum = cadd(sum, a[j - 1]);
  }
  v[0] = sum;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double2 A = x0, B = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const int e = (j * k) % P;
      A.x = fma(K::c(e), a[j - 1].x, A.x);
      A.y = fma(K::c(e), a[j - 1].y, A.y);
      B.x = fma(K::s(e), b[j - 1].x, B.x);
      B.y = fma(K::s(e), b[j - 1].y, B.y);
    }
    const double2 sb = mul_si<S>(B);
    v[k] = cadd(A, sb);
    v[P - k] = csub(A, sb);
  }
}

// Same transform, register-lean: the symmetric pairs overwrite the inputs in
// place (v[j] <- a_j, v[P-j] <- b_j) and every output pair is stored to the
// padded smem line as soon as it is formed (2P + 6 live doubles, not 4P).
template <int P, int S, int L>
__device__ __forceinline__ void dft_odd_store(double2* v, double2* buf, int base, int Ns) {
  constexpr int H = (P - 1) / 2;
  using K = OddConst<P>;
  const double2 x0 = v[0];
  double2 sum = x0;
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    const double2 a = cadd(v[j], v[P - j]);
    const double2 b = csub(v[j], v[P - j]);
    v[j] = a;
    v[P - j] = b;
    sum = cadd(sum, a);
  }
  buf[pad<L>(base)] = sum;
#pragma unroll
  for (int k = 1; k <= H; ++k) {
    double2 A = x0, B = make_double2(0.0, 0.0);
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      const int e = (j * k) % P;
      A.x = fma(K::c(e), v[j].x, A.x);
      A.y = fma(K::c(e), v[j].y, A.y);
      B.x = fma(K::s(e), v[P - j].x, B.x);
      B.y = fma(K::s(e), v[P - j].y, B.y);
    }
    const double2 sb = mul_si<S>(B);
    buf[pad<L>(base + k * Ns)] = cadd(A, sb);
    buf[pad<L>(base + (P - k) * Ns)] = csub(A, sb);
  }
}

template <int R, int S>
__device__ __forceinline__ void dft(double2* v) {
  if constexpr (R == 2) dft2<S>(v);
  else if constexpr (R == 4) dft4<S>(v[0], v[1], v[2], v[3]);
  else if constexpr (R == 8) dft8<S>(v);
  else if constexpr (R == 3) dft3<S>(v);
  else if constexpr (R == 6) dft6<S>(v);
  else if constexpr (R == 5) dft5<S>(v);
  else if constexpr (R == 9) dft9<S>(v);
  else if constexpr (R == 15) dft15<S>(v);
  else dft_odd<R, S>(v);
}

// v[r] *= W^r (S < 0) or conj(W^r) (S > 0), r = 1..R-1, with the powers formed
// on the fly from a window of four: w_r = w_{r-4} w_4 for r > 4 (product depth
// <= r/4 + 2, a few ulp), so at most five twiddles are live instead of R-1.
template <int R, int S>
__device__ __forceinline__ void apply_twiddles(double2* v, double2 w1) {
  double2 win[4];
  win[0] = w1;
  win[1] = cmul(w1, w1);
  win[2] = cmul(win[1], w1);
  win[3] = cmul(win[1], win[1]);
  const double2 w4 = win[3];
#pragma unroll
  for (int r = 1; r < R; ++r) {
    if (r > 4) win[(r - 1) & 3] = cmul(win[(r - 1) & 3], w4);
    v[r] = S < 0 ? cmul(v[r], win[(r - 1) & 3]) : cmulc(v[r], win[(r - 1) & 3]);
  }
}

// Barrier of the threads working on one line: id 0 = the whole CTA
// (__syncthreads), id > 0 = named barrier over the line's T threads (whole
// warps), so the lines of a CTA run their stages independently.
__device__ __forceinline__ void line_sync(int id, int nthreads) {
  if (id == 0) {
    __syncthreads();
  } else {
    asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(nthreads) : "memory");
  }
}

// Default input of a stage: the line itself.
struct LineIn {};

// One Stockham stage on a padded in-smem line.  With an input functor fin
// (first stage only), v = fin(i) replaces the load of natural index i: the
// producer of the line (pointwise spectrum product, residual, extension) is
// folded into the stage's loads instead of a separate smem pass + barrier.
// fin may read the line itself: every load precedes the stage's barrier.
template <int L, int Ns, int R, int S, int T, typename F = LineIn>
__device__ __forceinline__ void stage(double2* buf, const double2* __restrict__ tw, int t, int bar = 0,
                                      F fin = F()) {
  constexpr bool FIN = !std::is_same<F, LineIn>::value;
  constexpr int NB = L / R;
  constexpr int PER = (NB + T - 1) / T;
  double2 v[PER][R];
  double2 w1[PER];
  // base twiddles first: their (L1/L2) latency overlaps the smem loads and
  // the barrier; the powers are formed per butterfly after it (registers)
  if constexpr (Ns > 1) {
    constexpr int step = L / (Ns * R);
#pragma unroll
    for (int i = 0; i < PER; ++i) {
      const int b = t + i * T;
      if (NB % T == 0 || b < NB) w1[i] = tw[(b % Ns) * step];
    }
  }
  // padded addresses linear in r (base + immediate offsets) when the stride
  // is a multiple of the padding period (or L is odd: no padding)
  constexpr bool LIN_IN = (L & 1) || (NB % 8 == 0);
  constexpr int SIN = (L & 1) ? NB : NB + NB / 8;
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int b = t + i * T;
    if (NB % T == 0 || b < NB) {
      if constexpr (FIN) {
#pragma unroll
        for (int r = 0; r < R; ++r) v[i][r] = fin(b + r * NB);
      } else if constexpr (LIN_IN) {
        const double2* src = buf + pad<L>(b);
#pragma unroll
        for (int r = 0; r < R; ++r) v[i][r] = src[r * SIN];
      } else {
#pragma unroll
        for (int r = 0; r < R; ++r) v[i][r] = buf[pad<L>(b + r * NB)];
      }
    }
  }
  line_sync(bar, T);
#pragma unroll
  for (int i = 0; i < PER; ++i) {
    const int b = t + i * T;
    if (NB % T == 0 || b < NB) {
      const int k = b % Ns;
      if constexpr (Ns > 1) apply_twiddles<R, S>(v[i], w1[i]);
      const int base = (b / Ns) * Ns * R + k;
      if constexpr (R >= 7 && (R & 1) && R != 9 && R != 15) {
        dft_odd_store<R, S, L>(v[i], buf, base, Ns);
      } else {
        dft<R, S>(v[i]);
        // Ns % 8 == 0: pad(base + r Ns) = pad(base) + r Ns 9/8; Ns == 1, R == 8:
        // pad(8b + r) = 9b + r
        constexpr bool LIN_OUT = (L & 1) || (Ns % 8 == 0) || (Ns == 1 && R == 8);
        constexpr int SOUT = (L & 1) ? Ns : (Ns % 8 == 0 ? Ns + Ns / 8 : 1);
        if constexpr (LIN_OUT) {
          double2* dst = buf + pad<L>(base);
#pragma unroll
          for (int r = 0; r < R; ++r) dst[r * SOUT] = v[i][r];
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) buf[pad<L>(base + r * Ns)] = v[i][r];
        }
      }
    }
  }
  line_sync(bar, T);
}

// Output pairs K0..K1 (compile-time) of one odd-prime butterfly whose
// symmetric pairs a_j = v_j + v_{R-j}, b_j = v_j - v_{R-j} sit in shared
// memory at the butterfly's input slots (j, R-j): one sweep over j feeds all
// KP pairs (4 KP independent FMA chains, constants as immediate operands).
// The outputs stay in registers (out[2u] = X_{K0+u}, out[2u+1] = X_{R-K0-u}).
template <int R, int S, int L, int K0, int K1>
__device__ __forceinline__ void odd_pairs_smem(const double2* buf, int b, int NB, double2 x0, double2* out,
                                               double2* sum = nullptr) {
  using K = OddConst<R>;
  constexpr int H = (R - 1) / 2;
  constexpr int KP = K1 - K0 + 1;
  double2 A[KP], B[KP];
#pragma unroll
  for (int u = 0; u < KP; ++u) {
    A[u] = x0;
    B[u] = make_double2(0.0, 0.0);
  }
#pragma unroll
  for (int j = 1; j <= H; ++j) {
    const double2 a = buf[pad<L>(b + j * NB)], c = buf[pad<L>(b + (R - j) * NB)];
    if (sum) *sum = cadd(*sum, a);
#pragma unroll
    for (int u = 0; u < KP; ++u) {
      const int e = (j * (K0 + u)) % R;
      A[u].x = fma(K::c(e), a.x, A[u].x);
      A[u].y = fma(K::c(e), a.y, A[u].y);
      B[u].x = fma(K::s(e), c.x, B[u].x);
      B[u].y = fma(K::s(e), c.y, B[u].y);
    }
  }
#pragma unroll
  for (int u = 0; u < KP; ++u) {
    const double2 sb = mul_si<S>(B[u]);
    out[2 * u] = cadd(A[u], sb);
    out[2 * u + 1] = csub(A[u], sb);
  }
}

template <int R, int S, int L, int H, int P, int Q, int KPM>
__device__ __forceinline__ void odd_pairs_smem_dispatch(int part, const double2* buf, int b, int NB, double2 x0,
                                                        double2* out, double2* sum0 = nullptr) {
  if constexpr (Q < P) {
    if (part == Q) {
      odd_pairs_smem<R, S, L, 1 + (Q * H) / P, ((Q + 1) * H) / P>(buf, b, NB, x0, out, Q == 0 ? sum0 : nullptr);
      return;
    }
    odd_pairs_smem_dispatch<R, S, L, H, P, Q + 1, KPM>(part, buf, b, NB, x0, out, sum0);
  }
}

template <int R, int S, int L, int H, int P, int Q>
__device__ __forceinline__ void odd_pairs_store_dispatch(int part, const double2* out, double2* buf, int base,
                                                         int Ns) {
  if constexpr (Q < P) {
    if (part == Q) {
      constexpr int K0 = 1 + (Q * H) / P, K1 = ((Q + 1) * H) / P;
#pragma unroll
      for (int u = 0; u <= K1 - K0; ++u) {
        buf[pad<L>(base + (K0 + u) * Ns)] = out[2 * u];
        buf[pad<L>(base + (R - K0 - u) * Ns)] = out[2 * u + 1];
      }
      return;
    }
    odd_pairs_store_dispatch<R, S, L, H, P, Q + 1>(part, out, buf, base, Ns);
  }
}

// CTA-wide stage for a large odd prime R (>= 17) on G lines at once: the
// G * NB butterflies (NB = L/R is small, e.g. 33 for 1023 = 31*33) are packed
// densely over a warp-aligned slot range of NBp threads, replicated P times
// (P = CTA threads / NBp).  Register-lean three-phase form: (1) replica 0
// twiddles its butterfly's inputs and folds them into the symmetric pairs in
// place (a_j at slot j, b_j at slot R-j) and keeps X_0; (2) every replica p
// sweeps the pairs once for its output range (pH/P, (p+1)H/P], results in
// registers; (3) after a barrier the outputs go to the Stockham positions.
// No thread holds the R inputs at once, so the stage needs ~4(H/P) + O(1)
// live complex values instead of R + accumulators.
// Twiddle-free (first) large-prime stage whose G*NB butterflies do not fill
// whole warps (1023 = 31*33 on two lines: 66 = 2*32 + 2).  The padded form
// above runs P replicas of ceil(66/32) = 3 warps, two of them with 2 of 32
// lanes busy but still issuing every FMA of the sweep (a third of the stage's
// FP64 issue).  Here the P replicas cover only the NBf = 64 butterflies that
// fill warps; one extra warp takes the REM leftovers with one output pair per
// lane (REM*H <= 32 lanes), its cos/sin weights read from a shared-memory copy
// of the constant table (runtime k), so its sweep costs H FMA quadruples.
template <int L, int R, int S, int G, int PL, int NTH>
struct OddSplit {
  static constexpr int NB = L / R, H = (R - 1) / 2;
  static constexpr int NBt = G * NB, NBf = NBt / 32 * 32, REM = NBt - NBf;
  static constexpr int P0 = NBf > 0 ? (NTH - 32) / NBf : 0;
  static constexpr int P = P0 > H ? H : P0;
  static constexpr bool ok = REM > 0 && NBf > 0 && P >= 1 && REM * H <= 32 && NTH % 32 == 0;
};

template <int L, int R, int S, int G, int PL, int NTH>
__device__ __forceinline__ void stage_odd_cta_split(double2* sm, int tid) {
  using Z = OddSplit<L, R, S, G, PL, NTH>;
  using K = OddConst<R>;
  constexpr int NB = Z::NB, H = Z::H, NBf = Z::NBf, P = Z::P;
  constexpr int KPM = (H + P - 1) / P;
  __shared__ double2 ocs[R];  // (cos, sin)(2 pi e / R)
  if (tid < R) ocs[tid] = make_double2(K::c(tid), K::s(tid));
  const int part = tid / NBf;  // warp-uniform (NBf % 32 == 0)
  const bool mainp = part < P;
  const int lane = tid - P * NBf;
  const bool rem = lane >= 0 && lane < Z::REM * H;
  // main butterflies: slots 0 .. NBf-1; leftover lane: butterfly NBf + lane/H, pair k
  const int slot = mainp ? tid - part * NBf : (rem ? NBf + lane / H : 0);
  const int line = slot / NB;
  const int b = slot - line * NB;
  double2* buf = sm + line * PL;
  const int kr = rem ? 1 + lane % H : 0;
  // fold the symmetric pairs in place (a_j at slot j, b_j at slot R-j)
  if (mainp) {
    const int j0 = 1 + (part * H) / P, j1 = ((part + 1) * H) / P;
    for (int j = j0; j <= j1; ++j) {
      double2& vj = buf[pad<L>(b + j * NB)];
      double2& vm = buf[pad<L>(b + (R - j) * NB)];
      const double2 x = vj, y = vm;
      vj = cadd(x, y);
      vm = csub(x, y);
    }
  } else if (rem) {
    double2& vj = buf[pad<L>(b + kr * NB)];
    double2& vm = buf[pad<L>(b + (R - kr) * NB)];
    const double2 x = vj, y = vm;
    vj = cadd(x, y);
    vm = csub(x, y);
  }
  __syncthreads();
  double2 out[2 * KPM];
  double2 sum = make_double2(0.0, 0.0);
  if (mainp) {
    sum = buf[pad<L>(b)];
    odd_pairs_smem_dispatch<R, S, L, H, P, 0, KPM>(part, buf, b, NB, sum, out, &sum);
  } else if (rem) {
    const double2 x0 = buf[pad<L>(b)];
    double2 A = x0, B = make_double2(0.0, 0.0);
    sum = x0;
    int e = 0;
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      e += kr;
      e = e >= R ? e - R : e;  // (j * kr) mod R
      const double2 a = buf[pad<L>(b + j * NB)], c = buf[pad<L>(b + (R - j) * NB)];
      const double2 w = ocs[e];
      sum = cadd(sum, a);
      A.x = fma(w.x, a.x, A.x);
      A.y = fma(w.x, a.y, A.y);
      B.x = fma(w.y, c.x, B.x);
      B.y = fma(w.y, c.y, B.y);
    }
    const double2 sb = mul_si<S>(B);
    out[0] = cadd(A, sb);
    out[1] = csub(A, sb);
  }
  __syncthreads();
  const int base = b * R;  // Ns = 1
  if (mainp) {
    if (part == 0) buf[pad<L>(base)] = sum;
    odd_pairs_store_dispatch<R, S, L, H, P, 0>(part, out, buf, base, 1);
  } else if (rem) {
    if (kr == 1) buf[pad<L>(base)] = sum;
    buf[pad<L>(base + kr)] = out[0];
    buf[pad<L>(base + R - kr)] = out[1];
  }
  __syncthreads();
}

// FP64 tensor-core form of the twiddle-free (first) stage of a large odd
// prime R (29, 31: H + 1 = (R+1)/2 <= 16, so nothing pads beyond 16): after
// the in-place fold (a_j at slot j, b_j at slot R-j, x_0 at slot 0) the
// stage's G*NB butterflies are two small real GEMMs on all of them at once,
//   A[k][col] = sum_{j=0..H} Cw[k][j] * Aval[j][col],  Cw = [1 | cos(2 pi jk/R)]
//   B[k][col] = sum_{j=1..H} Sw[k][j] * Bval[j][col],  Sw = sin(2 pi jk/R)
// k = 0..H (row 0 of Cw is all ones: A[0] = X_0), col = 2 b + {re, im} of
// butterfly b (the fold keeps a butterfly's complex value contiguous, so a
// GEMM row j is the line's slot range [j NB, j NB + NB) read as doubles), and
// X_k = A_k + S i B_k, X_{R-k} = A_k - S i B_k.  mma.sync.m8n8k4.f64: M = 16
// (two m-tiles), K = 16 (four k-steps), N = 8 columns per tile; a warp task
// is one (line, n-tile, m-tile) with 8 DMMA (cos + sin), the weight
// fragments live in registers for the whole stage.  One DMMA is 256 FMAs, so
// the stage's 900 FMAs per butterfly issue as ~4 warp instructions instead of
// ~28 DFMA ones.  But the FP64 pipe is shared (DMMA + DFMA concurrently:
// 35.4 TF/s, profiles/r02_fp64_peak.json) and the tiles pad 116% of the
// useful FMAs, so the stage costs ~7% more pipe time than the DFMA sweep;
// measured A/B on C3 (profiles/r02_dmma_ab.md): transform class 92.7 vs 89.4
// ms/step, -2.7% overall.  Opt-in (-DDBX_DMMA_STAGE), not the default.
template <int L, int R, int S, int G, int PL, int NTH>
struct OddDmma {
  static constexpr int NB = L / R, H = (R - 1) / 2;
  static constexpr int NCOL = 2 * NB, NTILE = (NCOL + 7) / 8;
  static constexpr int TASKS = G * NTILE * 2;           // (line, n-tile, m-tile)
  static constexpr int NW = NTH / 32;
  static constexpr int TPW = (TASKS + NW - 1) / NW;     // tasks per warp
  static constexpr bool ok = H + 1 <= 16 && H >= 14 && NTH % 32 == 0 && (L & 1);
};

__device__ __forceinline__ void dmma_f64(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

template <int L, int R, int S, int G, int PL, int NTH>
__device__ __forceinline__ void stage_odd_cta_dmma(double2* sm, int tid) {
  using Z = OddDmma<L, R, S, G, PL, NTH>;
  using K = OddConst<R>;
  constexpr int NB = Z::NB, H = Z::H, NTILE = Z::NTILE, TPW = Z::TPW, NW = Z::NW;
  __shared__ double2 ocs[R];  // (cos, sin)(2 pi e / R)
  if (tid < R) ocs[tid] = make_double2(K::c(tid), K::s(tid));
  // fold every butterfly's symmetric pairs in place
  for (int e = tid; e < G * NB * H; e += NTH) {
    const int line = e / (NB * H), r = e - line * (NB * H);
    const int j = 1 + r / NB, b = r - (j - 1) * NB;
    double2* buf = sm + line * PL;
    double2& vj = buf[b + j * NB];
    double2& vm = buf[b + (R - j) * NB];
    const double2 x = vj, y = vm;
    vj = cadd(x, y);
    vm = csub(x, y);
  }
  __syncthreads();
  const int lane = tid & 31, warp = tid >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  // weight fragments (A operand: row k = 8 mt + gid, col j = 4 ks + tig)
  double cw[2][4], sw[2][4];
#pragma unroll
  for (int mt = 0; mt < 2; ++mt)
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      const int k = 8 * mt + gid, j = 4 * ks + tig;
      const bool in = k <= H && j <= H;
      const double2 w = ocs[(j * k) % R];
      cw[mt][ks] = in ? (j == 0 ? 1.0 : w.x) : 0.0;
      sw[mt][ks] = in && j > 0 ? w.y : 0.0;
    }
  double res[TPW][4];
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    const int task = warp + u * NW;  // warp-uniform
    res[u][0] = res[u][1] = res[u][2] = res[u][3] = 0.0;
    if (task < Z::TASKS) {
      const int mt = task & 1, tl = task >> 1;
      const int line = tl / NTILE, nt = tl - line * NTILE;
      const double* bd = reinterpret_cast<const double*>(sm + line * PL);
      const int col = 8 * nt + gid;         // B operand column of this lane
      const bool cv = col < 2 * NB;
      double ac[2] = {0.0, 0.0}, bs[2] = {0.0, 0.0};
#pragma unroll
      for (int ks = 0; ks < 4; ++ks) {
        const int j = 4 * ks + tig;          // B operand row: j <= 15
        const bool jv = cv && j <= H;
        const double av = jv ? bd[2 * j * NB + col] : 0.0;                       // x_0 / a_j
        const double bv = jv && j > 0 ? bd[2 * (R - j) * NB + col] : 0.0;        // b_j
        dmma_f64(ac, mt ? cw[1][ks] : cw[0][ks], av);
        dmma_f64(bs, mt ? sw[1][ks] : sw[0][ks], bv);
      }
      res[u][0] = ac[0]; res[u][1] = ac[1]; res[u][2] = bs[0]; res[u][3] = bs[1];
    }
  }
  __syncthreads();  // every butterfly's inputs are consumed before the in-place outputs
#pragma unroll
  for (int u = 0; u < TPW; ++u) {
    const int task = warp + u * NW;
    if (task < Z::TASKS) {
      const int mt = task & 1, tl = task >> 1;
      const int line = tl / NTILE, nt = tl - line * NTILE;
      const int k = 8 * mt + gid;            // accumulator row
      const int b = 4 * nt + tig;            // accumulator cols (2b, 2b+1) = butterfly b
      if (k <= H && b < NB) {
        double2* buf = sm + line * PL;
        const double2 A = make_double2(res[u][0], res[u][1]);
        const double2 sb = mul_si<S>(make_double2(res[u][2], res[u][3]));
        const int base = b * R;                // Ns = 1
        if (k == 0) {
          buf[base] = A;
        } else {
          buf[base + k] = cadd(A, sb);
          buf[base + R - k] = csub(A, sb);
        }
      }
    }
  }
  __syncthreads();
}

template <int L, int Ns, int R, int S, int G, int PL, int NTH>
__device__ __forceinline__ void stage_odd_cta(double2* sm, const double2* __restrict__ tw, int tid) {
#ifdef DBX_DMMA_STAGE
  if constexpr (Ns == 1 && OddDmma<L, R, S, G, PL, NTH>::ok) {
    stage_odd_cta_dmma<L, R, S, G, PL, NTH>(sm, tid);
    return;
  }
#endif
#ifndef DBX_NO_ODD_SPLIT
  if constexpr (Ns == 1 && OddSplit<L, R, S, G, PL, NTH>::ok) {
    stage_odd_cta_split<L, R, S, G, PL, NTH>(sm, tid);
    return;
  }
#endif
  constexpr int NB = L / R;
  constexpr int H = (R - 1) / 2;
  constexpr int NBp = (G * NB + 31) / 32 * 32;
  constexpr int P0 = NTH / NBp;
  constexpr int P = P0 < 1 ? 1 : (P0 > H ? H : P0);
  constexpr int KPM = (H + P - 1) / P;
  const int part = tid / NBp;                 // warp-uniform
  const int slot = tid - part * NBp;
  const bool act = part < P && slot < G * NB;
  const int line = act ? slot / NB : 0;
  const int b = act ? slot - line * NB : 0;
  double2* buf = sm + line * PL;
  const int k = b % Ns;
  double2 sum = make_double2(0.0, 0.0);
  if constexpr (Ns == 1) {
    // no twiddles: every replica folds its own share of the pairs; replica 0
    // accumulates X_0 while it sweeps the pairs in phase 2
    if (act) {
      const int j0 = 1 + (part * H) / P, j1 = ((part + 1) * H) / P;
      for (int j = j0; j <= j1; ++j) {
        double2& vj = buf[pad<L>(b + j * NB)];
        double2& vm = buf[pad<L>(b + (R - j) * NB)];
        const double2 x = vj, y = vm;
        vj = cadd(x, y);
        vm = csub(x, y);
      }
    }
  } else if (act && part == 0) {
    {
      // twiddle the inputs in place (r = 1..R-1), powers by the window scheme
      constexpr int step = L / (Ns * R);
      const double2 w1 = tw[k * step];
      double2 win[4];
      win[0] = w1;
      win[1] = cmul(w1, w1);
      win[2] = cmul(win[1], w1);
      win[3] = cmul(win[1], win[1]);
      const double2 w4 = win[3];
#pragma unroll
      for (int r = 1; r < R; ++r) {
        if (r > 4) win[(r - 1) & 3] = cmul(win[(r - 1) & 3], w4);
        double2& x = buf[pad<L>(b + r * NB)];
        x = S < 0 ? cmul(x, win[(r - 1) & 3]) : cmulc(x, win[(r - 1) & 3]);
      }
    }
    sum = buf[pad<L>(b)];
#pragma unroll
    for (int j = 1; j <= H; ++j) {
      double2& vj = buf[pad<L>(b + j * NB)];
      double2& vm = buf[pad<L>(b + (R - j) * NB)];
      const double2 x = vj, y = vm;
      const double2 a = cadd(x, y);
      vj = a;
      vm = csub(x, y);
      sum = cadd(sum, a);
    }
  }
  __syncthreads();
  double2 out[2 * KPM];
  if constexpr (Ns == 1) {
    if (act) {
      sum = buf[pad<L>(b)];
      odd_pairs_smem_dispatch<R, S, L, H, P, 0, KPM>(part, buf, b, NB, sum, out, &sum);
    }
  } else if (act) {
    odd_pairs_smem_dispatch<R, S, L, H, P, 0, KPM>(part, buf, b, NB, buf[pad<L>(b)], out);
  }
  __syncthreads();
  if (act) {
    const int base = (b / Ns) * Ns * R + k;
    if (part == 0) buf[pad<L>(base)] = sum;
    odd_pairs_store_dispatch<R, S, L, H, P, 0>(part, out, buf, base, Ns);
  }
  __syncthreads();
}

template <int L, int Ns, int S, int T>
__device__ __forceinline__ void run_stages(double2* buf, const double2* __restrict__ tw, int t, int bar) {
  if constexpr (Ns < L) {
    constexpr int R = next_radix(L / Ns);
    static_assert(R != 0, "FFT length must factor into {2,3,4,5,8} and odd primes <= 31");
    stage<L, Ns, R, S, T>(buf, tw, t, bar);
    run_stages<L, Ns * R, S, T>(buf, tw, t, bar);
  }
}

// CTA-wide variant: G lines of PL (padded) elements starting at sm, T threads
// per line; thread tid = g*T + t.  Large odd-prime stages run packed across
// the lines (stage_odd_cta), the rest per line.
template <int L, int Ns, int S, int T, int G, int PL>
__device__ __forceinline__ void run_stages_cta(double2* sm, const double2* __restrict__ tw, int tid) {
  if constexpr (Ns < L) {
    constexpr int R = next_radix(L / Ns);
    static_assert(R != 0, "FFT length must factor into {2,3,4,5,8} and odd primes <= 31");
    if constexpr (R >= 17 && (R & 1) && G * (L / R) <= G * T) {
      if constexpr (Ns > 1) __syncthreads();  // threads read other lines here
      stage_odd_cta<L, Ns, R, S, G, PL, G * T>(sm, tw, tid);
    } else {
      const int g = tid / T;
      stage<L, Ns, R, S, T>(sm + g * PL, tw, tid - g * T, G > 1 ? 1 + g : 0);
    }
    PH(40 + (Ns == 1 ? 0 : (Ns * R == L ? 2 : 1)))  // DST FFT stage (first / middle / last)
    run_stages_cta<L, Ns * R, S, T, G, PL>(sm, tw, tid);
  }
}

template <int L, int S, int T, int G>
__device__ __forceinline__ void fft_cta(double2* sm, const double2* __restrict__ tw, int tid) {
  static_assert(supported(L), "unsupported FFT length");
  run_stages_cta<L, 1, S, T, G, padded_len(L)>(sm, tw, tid);
}

// In-place unnormalised FFT of one padded line; S = -1 forward, +1 inverse.
// Every thread of the line's group must call it; bar = 0 synchronises the
// whole CTA, bar > 0 only the line's T threads (named barrier `bar`).
template <int L, int S, int T>
__device__ __forceinline__ void fft(double2* buf, const double2* __restrict__ tw, int t, int bar = 0) {
  static_assert(supported(L), "unsupported FFT length");
  run_stages<L, 1, S, T>(buf, tw, t, bar);
}

// As fft, with the first stage's inputs produced by fin(natural index) (see
// stage); the line's previous contents may be read by fin.
template <int L, int S, int T, typename F>
__device__ __forceinline__ void fft_in(double2* buf, const double2* __restrict__ tw, int t, int bar, F fin) {
  static_assert(supported(L), "unsupported FFT length");
  constexpr int R = next_radix(L);
  stage<L, 1, R, S, T>(buf, tw, t, bar, fin);
  run_stages<L, R, S, T>(buf, tw, t, bar);
}


// ---------------------------------------------------------------------------
// In-place Cooley-Tukey (no autosort) for convolution cores (Rader, Bluestein):
// forward = decimation in frequency from natural order to digit-reversed order
// (radix.h ct_freq_of_pos), the pointwise kernel product in that order (the
// host permutes the kernel spectrum), inverse = decimation in time from
// digit-reversed back to natural order.  Each butterfly reads and writes the
// same R slots, so a thread finishes one butterfly (load, DFT, twiddles,
// store) before it loads the next: one barrier per stage and R live complex
// values per thread, against the Stockham stage's two barriers and PER x R
// registers.  The last forward level, the kernel product and the first
// inverse level act on the same contiguous R-blocks and run as one pass.

// Butterflies a thread keeps in flight per pass (all loads of the group are
// issued before the first DFT): about 16 complex values, so short radices get
// load-level parallelism and long ones stay within the register budget.
#ifndef DBX_CT_VALS
#define DBX_CT_VALS 16
#endif
template <int R, int NB, int T>
__host__ __device__ constexpr int ct_unroll() {
  constexpr int u = DBX_CT_VALS / R < 1 ? 1 : DBX_CT_VALS / R;
  constexpr int per = (NB + T - 1) / T;
  return u < per ? u : per;
}

// Forward level with block size Ls (m = Ls/R): y_k = DFT_R(x_{j + r m}),
// y_k *= W_Ls^{j k}.  DIR = -1; the inverse level (DIR = +1, transpose of the
// forward one, conjugated) multiplies by conj W_Ls^{j k} first, then runs the
// unnormalised inverse DFT_R.
template <int L, int Ls, int T, int DIR>
__device__ __forceinline__ void ct_level(double2* buf, const double2* __restrict__ tw, int t, int bar) {
  constexpr int R = ct_radix(Ls), m = Ls / R, NB = L / R;
  static_assert(R != 0, "unsupported FFT length");
  constexpr int U = ct_unroll<R, NB, T>();
#pragma unroll 1
  for (int b0 = t; b0 < NB; b0 += U * T) {
    double2 v[U][R], w1[U];
    int base[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int beta = b0 + u * T;
      int blk = beta / m, j = beta - blk * m;
      if constexpr (ct_nopad(L) && m < 8 && m % 2 == 0 && Ls % 8 == 2) {
        // short blocks, unpadded line: a quarter warp takes 2 j's of 4 blocks
        // (slots blk Ls + j = 2 blk + j mod 8: eight distinct 16-byte bank
        // groups) instead of 8 consecutive butterflies (6 of one block + 2 of
        // the next: two groups hit twice); the blocks past the last multiple
        // of 4 keep the plain order
        constexpr int MAIN = (L / Ls) / 4 * 4 * m;
        if (beta < MAIN) {
          const int lo = beta & 7, rest = beta >> 3;
          const int bh = rest / (m / 2), jh = rest - bh * (m / 2);
          j = 2 * jh + (lo & 1);
          blk = 4 * bh + (lo >> 1);
        }
      }
      base[u] = blk * Ls + j;
      if (U == 1 || beta < NB) {
        w1[u] = tw[j * (L / Ls)];  // smem-staged or global table
#pragma unroll
        for (int r = 0; r < R; ++r) v[u][r] = buf[pad<L>(base[u] + r * m)];
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (U == 1 || b0 + u * T < NB) {
        if constexpr (DIR < 0) {
          dft<R, -1>(v[u]);
          apply_twiddles<R, -1>(v[u], w1[u]);
        } else {
          apply_twiddles<R, +1>(v[u], w1[u]);
          dft<R, +1>(v[u]);
        }
#pragma unroll
        for (int r = 0; r < R; ++r) buf[pad<L>(base[u] + r * m)] = v[u][r];
      }
    }
  }
  line_sync(bar, T);
}

template <int L, int Ls, int T>
__device__ __forceinline__ void ct_dif_levels(double2* buf, const double2* __restrict__ tw, int t, int bar) {
  if constexpr (Ls / ct_radix(Ls) > 1) {  // every level but the last (R-blocks)
    ct_level<L, Ls, T, -1>(buf, tw, t, bar);
    ct_dif_levels<L, Ls / ct_radix(Ls), T>(buf, tw, t, bar);
  }
}
template <int L, int Ls, int T>
__device__ __forceinline__ void ct_dit_levels(double2* buf, const double2* __restrict__ tw, int t, int bar) {
  if constexpr (Ls / ct_radix(Ls) > 1) {
    ct_dit_levels<L, Ls / ct_radix(Ls), T>(buf, tw, t, bar);
    ct_level<L, Ls, T, +1>(buf, tw, t, bar);
  }
}
// size of the innermost level's blocks (the last forward radix)
template <int L>
__host__ __device__ constexpr int ct_last_radix() {
  int Ls = L;
  while (Ls / ct_radix(Ls) > 1) Ls /= ct_radix(Ls);
  return Ls;
}

// Cyclic convolution core: buf <- IDFT(K .* DFT(buf)) with K the kernel
// spectrum in digit-reversed position order (kdr[p] = K_{ct_freq_of_pos(p)}),
// unnormalised inverse (the host folds 1/L into K).  x0 (may be null)
// receives DFT(buf)_0 (position 0, before the product).  bar as for fft().
// KT: kdr is element-major, kdr[r NB + b] (tables.cpp bctT): consecutive
// butterflies read consecutive addresses (one 512-byte row per warp load
// instead of 32 lanes R * 16 bytes apart).
#ifndef DBX_CT_KT
#define DBX_CT_KT 1
#endif
__host__ __device__ constexpr bool ct_kt(int L) { return DBX_CT_KT && ct_nopad(L); }
template <int L, int T, bool KT = false>
__device__ __forceinline__ void ct_convolve(double2* buf, const double2* __restrict__ tw,
                                            const double2* kdr, int t, int bar, double2* x0) {
  static_assert(supported(L), "unsupported FFT length");
  ct_dif_levels<L, L, T>(buf, tw, t, bar);
  constexpr int R = ct_last_radix<L>(), NB = L / R;
  constexpr int U = ct_unroll<R, NB, T>();
  // unpadded R-blocks with R = 2 mod 4 (slots R b + r): lanes 0-3 of each
  // group of 8 touch element r and lanes 4-7 element r ^ 1, so a quarter warp
  // covers all eight 16-byte bank groups (R b + r alone reaches only four)
  constexpr bool SWAP2 = ct_nopad(L) && R % 4 == 2 && T % 8 == 0;
  const int sel = (t >> 2) & 1;
#pragma unroll 1
  for (int b0 = t; b0 < NB; b0 += U * T) {
    double2 v[U][R];
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (U == 1 || b0 + u * T < NB) {
#pragma unroll
        if constexpr (SWAP2) {
#pragma unroll
          for (int r = 0; r < R; r += 2) {
            const double2 a = buf[(b0 + u * T) * R + (r ^ sel)], c = buf[(b0 + u * T) * R + (r ^ sel ^ 1)];
            v[u][r] = sel ? c : a;
            v[u][r + 1] = sel ? a : c;
          }
        } else {
          for (int r = 0; r < R; ++r) v[u][r] = buf[pad<L>((b0 + u * T) * R + r)];
        }
      }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int base = (b0 + u * T) * R;
      if (U == 1 || b0 + u * T < NB) {
        dft<R, -1>(v[u]);
        if (x0 && base == 0) *x0 = v[u][0];
#pragma unroll
        for (int r = 0; r < R; ++r) v[u][r] = cmul(v[u][r], KT ? kdr[r * NB + (b0 + u * T)] : kdr[base + r]);  // global or smem-staged
        dft<R, +1>(v[u]);
        if constexpr (SWAP2) {
#pragma unroll
          for (int r = 0; r < R; r += 2) {
            buf[base + (r ^ sel)] = sel ? v[u][r + 1] : v[u][r];
            buf[base + (r ^ sel ^ 1)] = sel ? v[u][r] : v[u][r + 1];
          }
        } else {
#pragma unroll
          for (int r = 0; r < R; ++r) buf[pad<L>(base + r)] = v[u][r];
        }
      }
    }
  }
  line_sync(bar, T);
  ct_dit_levels<L, L, T>(buf, tw, t, bar);
}

}  // namespace fft
}  // namespace dbx
