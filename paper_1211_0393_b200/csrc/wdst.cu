// wdst.cu — warp-owned packed DST-I for n = 1024 lines (N = 1023 = 31 * 33):
// the column half of D (T~ -> d -> T along columns of u) with no CTA barriers.
//
// Replaces (reference): sine1_forward / RODFT00 (transforms.hpp:114-121),
// ar_inverse then ar_forward (transforms.hpp:148-173) along the columns of
// tensor_map (transforms.hpp:179-192), and the Hadamard by d between them
// (filter_apply, spectral.hpp:161-165).
//
// One warp owns one packed DFT (two adjacent columns c, c+1 of one image) the
// whole way: global loads -> T~ fill -> DFT_1023 -> split + odd scan -> x d ->
// T fill -> DFT_1023 -> split + scan -> ramp epilogue -> row-major stores.
// Synchronisation is __syncwarp only, so the warps of an SM sit in different
// phases (loads of one overlap the FP64 DFTs of others) instead of the CTA
// lock-step of fused.cu's dst_tcols (a CTA barrier after every FFT stage).
//
// DFT_1023, Cooley-Tukey N = N2 * N1 with N1 = 33 (inner), N2 = 31, in-place
// on one padded smem line (slot(p) = p + p/32: the fill's per-lane contiguous
// runs hit distinct banks):
//   level 1  lane n2 < 31: x[31 n1 + n2], n1 < 33 -> in-register DFT-33 (3 x 11
//            Good-Thomas, no internal twiddles) -> * W_1023^{n2 k1} -> back to
//            the same slots (31 k1 + n2);
//   level 2  lane k1 < 32: the 31 contiguous slots 31 k1 + n2 -> in-register
//            DFT-31 (symmetric pairs, compile-time constants) -> X[k1 + 33 k2]
//            at slot 31 k1 + k2; the 33rd row (k1 = 32) is one output per lane.
// Packed real DST (spectral_common.cuh pk_fill / pk_split2 / odd_scans2): lane
// L owns output k in [32L, 32L+32), i.e. split pairs l in [16L, 16L+16): the
// odd-output prefix sum is 16 sequential adds plus one warp scan of lane totals
// (the same order as odd_scans2), and the mirrored fill operand N - k lives in
// lane 31 - L at index 31 - i (one shuffle per element).
#include <cuda_runtime.h>

#include "spectral_common.cuh"

namespace dbx {

namespace {

constexpr int kWN = 1023;     // DFT length
constexpr int kWLine = 1024;  // double2 slots per warp line
// per-warp line stride: one slot more than the line, so the CTA-cooperative
// reads of the 4 warps' outputs at the same k (64-byte row segments) hit 4
// different bank groups instead of one (1024 slots = 16 KB = 0 mod 128 B)
#ifndef DBX_WSTRIDE_PAD
#define DBX_WSTRIDE_PAD 2
#endif
constexpr int kWStride = kWLine + DBX_WSTRIDE_PAD;
constexpr int kWWarps = 4;    // warps (column pairs) per CTA
// CTAs per SM the register budget is sized for: 2 -> up to 255 registers (the
// DFT-31 row keeps 30 folded values + 30 constants live), 3 -> 168 (spills)
// Component-split DFT (-DDBX_WDST_RI=1, 168 registers, 12 warps/SM): measured
// 0.819 ms per C3 launch vs 0.762 for the complex-per-lane form at 8 warps/SM
// (and 0.794 for the split form at 8 warps) — the partner shuffles cost more
// than the extra occupancy buys.  Off by default.
#ifndef DBX_WDST_RI
#define DBX_WDST_RI 0
#endif
#ifndef DBX_WDST_MINB
#define DBX_WDST_MINB (DBX_WDST_RI ? 3 : 2)
#endif
// L2 prefetch (cp.async.bulk.prefetch.L2) of the input lines of the CTA this
// many resident waves ahead (0 = off)
#ifndef DBX_WDST_CTA_STORE
#define DBX_WDST_CTA_STORE 1
#endif
constexpr bool kWdstCtaStore = DBX_WDST_CTA_STORE != 0;
// warp-owned kernels for 256-point lines (C1); -DDBX_W255=0 keeps the CTA
// lock-step fused kernels there (A/B)
#ifndef DBX_W255
#define DBX_W255 1
#endif
constexpr bool kW255 = DBX_W255 != 0;
#ifndef DBX_WDST_PREFETCH
#define DBX_WDST_PREFETCH 0
#endif
// level-1 twiddles from the transposed table BlueTables::tw1t ([k1][lane]: one
// contiguous 512-byte row per warp load) instead of the strided gather
// tw[lane * k1] (up to 31 cache lines per load); -DDBX_TW1T=0 for the A/B
#ifndef DBX_TW1T
#define DBX_TW1T 1
#endif
// packed-DST fills in level-1 geometry, mirrors by shuffle (wfill_pre): the
// fill's store pass and level 1's load pass of every DFT_1023 are skipped at
// the price of 132 shuffles per DFT.  Opt-in (-DDBX_WPRE=1): parity green but
// measured slower (transform class 67.4 vs 64.1 ms/step, profiles/r02_wpre_ab.txt)
#ifndef DBX_WPRE
#define DBX_WPRE 0
#endif
// the cooperative 33rd level-2 row split between the lanes k2 (cosine sums)
// and 31 - k2 (sine sums): half its FP64 work and twiddle bytes
#ifndef DBX_WROW33_SPLIT
#define DBX_WROW33_SPLIT 1
#endif

// Two layouts share a warp's line.  DFT data at slot p (level 1 reads lanes at
// consecutive p, level 2 lanes at stride 31: both hit 8 distinct 16-byte bank
// groups per quarter warp).  Split outputs k at oslot(k) = k ^ ((k >> 5) & 7):
// the split writes lanes at stride 32 (k = 32 L + i), which the XOR spreads
// over the bank groups, and the fills / epilogue read lanes at consecutive k,
// which it keeps conflict-free.  Every change of layout is read-all, syncwarp,
// write-all.
__device__ __forceinline__ int wslot(int p) { return p; }
__device__ __forceinline__ int oslot(int k) { return k ^ ((k >> 5) & 7); }

// cos / sin(2 pi e / P) read through the half-period symmetry c(e) = c(P-e),
// s(e) = -s(P-e): with e compile-time after unrolling, a DFT-P needs only the
// (P-1)/2 + (P-1)/2 distinct constants in registers (negation folds into the
// DFMA operand), not P-1 + P-1.
template <int P>
__device__ __forceinline__ double ccs(int e) {
  return fft::OddConst<P>::c(e <= P / 2 ? e : P - e);
}
template <int P>
__device__ __forceinline__ double scs(int e) {
  return e <= P / 2 ? fft::OddConst<P>::s(e) : -fft::OddConst<P>::s(P - e);
}
// Level-2 row k1 lives at row position (k1 + kWRot) mod 33 (level 1 stores it
// there; position 32 is the cooperative row): with kWRot = 17 the split's
// loads (lanes 16 pairs apart) cost 156 instead of 280 wavefronts per DFT
// (128 ideal; rotation 0 puts lanes L and L + 1 in the same 16-byte bank group)
#ifndef DBX_WROT
#define DBX_WROT 17
#endif
constexpr int kWRot = DBX_WROT;
static_assert(!DBX_WDST_RI || DBX_WROT == 0, "the component-split DFT keeps the unrotated rows");
__host__ __device__ constexpr int wrow(int k1) { return (k1 + kWRot) % 33; }
// slot of DFT output frequency l after level 2 (k1 = l mod 33, k2 = l / 33)
__device__ __forceinline__ int wpos(int l) {
  const int k2 = l / 33, k1 = l - 33 * k2;
  return 31 * k1 + k2 + (k1 < 33 - kWRot ? 31 * kWRot : 31 * (kWRot - 33));
}

// Level-1 row of lane n2: in-register DFT-33 = 3 x 11 prime factor (input
// n = (11 a + 3 b) mod 33, output k1 = (22 ka + 12 kb) mod 33), each output
// twiddled by W_1023^{n2 k1} and stored to slot 31 k1 + n2 as soon as it is
// formed (register-lean: the DFT-3s run in place, the DFT-11 of group ka
// folds its inputs in place and emits its outputs pair by pair).
__device__ __forceinline__ void level1_row(double2* buf, const double2* __restrict__ tw, int lane, double2* v) {
  constexpr int S = -1;
#pragma unroll
  for (int b = 0; b < 11; ++b) {
    double2 t[3] = {v[(3 * b) % 33], v[(11 + 3 * b) % 33], v[(22 + 3 * b) % 33]};
    fft::dft3<S>(t);
    v[(3 * b) % 33] = t[0];
    v[(11 + 3 * b) % 33] = t[1];
    v[(22 + 3 * b) % 33] = t[2];
  }
  auto put = [&](int k1, double2 x) {
#if DBX_TW1T
    if (k1 != 0) x = fft::cmul(x, __ldg(tw + 32 * k1 + lane));  // tw = tw1t: [k1][lane], one 512-byte row per load
#else
    if (k1 != 0) x = fft::cmul(x, __ldg(tw + lane * k1));  // n2 k1 <= 990
#endif
    buf[31 * wrow(k1) + lane] = x;
  };
#pragma unroll
  for (int ka = 0; ka < 3; ++ka) {
    double2* u[11];
#pragma unroll
    for (int b = 0; b < 11; ++b) u[b] = &v[(11 * ka + 3 * b) % 33];
    const double2 x0 = *u[0];
    double2 sum = x0;
#pragma unroll
    for (int j = 1; j <= 5; ++j) {
      const double2 p = cadd(*u[j], *u[11 - j]), m = csub(*u[j], *u[11 - j]);
      *u[j] = p;
      *u[11 - j] = m;
      sum = cadd(sum, p);
    }
    put((22 * ka) % 33, sum);
#pragma unroll
    for (int k = 1; k <= 5; ++k) {
      double2 A = x0, B = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 1; j <= 5; ++j) {
        const int e = (j * k) % 11;
        A.x = fma(ccs<11>(e), u[j]->x, A.x);
        A.y = fma(ccs<11>(e), u[j]->y, A.y);
        B.x = fma(scs<11>(e), u[11 - j]->x, B.x);
        B.y = fma(scs<11>(e), u[11 - j]->y, B.y);
      }
      const double2 sb = fft::mul_si<S>(B);
      put((22 * ka + 12 * k) % 33, cadd(A, sb));
      put((22 * ka + 12 * (11 - k)) % 33, csub(A, sb));
    }
  }
}

__device__ __forceinline__ void wdft1023_tail(double2* buf, const double2* __restrict__ tw, int lane);
// Forward DFT_1023 of one warp's line (S = -1), in place; tw[e] = W_1023^e.
__device__ __forceinline__ void wdft1023(double2* buf, const double2* __restrict__ tw, int lane) {
  constexpr int S = -1;
  if (lane < 31) {
    double2 v[33];
#pragma unroll
    for (int n1 = 0; n1 < 33; ++n1) v[n1] = buf[wslot(31 * n1 + lane)];
    level1_row(buf, tw, lane, v);
  }
  __syncwarp();
  wdft1023_tail(buf, tw, lane);
}

// levels 2 and the cooperative 33rd row of DFT_1023 (after level 1's stores + __syncwarp)
__device__ __forceinline__ void wdft1023_tail(double2* buf, const double2* __restrict__ tw, int lane) {
  constexpr int S = -1;
  {
    // own row k1 = lane: 31 contiguous slots, outputs back in place
    const int base = 31 * lane;
    double2 v[31];
#pragma unroll
    for (int j = 0; j < 31; ++j) v[j] = buf[wslot(base + j)];
    const double2 x0 = v[0];
    double2 sum = x0;
#pragma unroll
    for (int j = 1; j <= 15; ++j) {
      const double2 a = cadd(v[j], v[31 - j]), b = csub(v[j], v[31 - j]);
      v[j] = a;
      v[31 - j] = b;
      sum = cadd(sum, a);
    }
    buf[wslot(base)] = sum;
#pragma unroll
    for (int k = 1; k <= 15; ++k) {
      double2 A = x0, B = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 1; j <= 15; ++j) {
        const int e = (j * k) % 31;
        A.x = fma(ccs<31>(e), v[j].x, A.x);
        A.y = fma(ccs<31>(e), v[j].y, A.y);
        B.x = fma(scs<31>(e), v[31 - j].x, B.x);
        B.y = fma(scs<31>(e), v[31 - j].y, B.y);
      }
      const double2 sb = fft::mul_si<S>(B);
      buf[wslot(base + k)] = cadd(A, sb);
      buf[wslot(base + 31 - k)] = csub(A, sb);
    }
  }
  // row k1 = 32 (slots 992..1022, untouched by the own rows): lane k2 < 31
  // forms X[32 + 33 k2] = sum_n2 Y[32][n2] W_31^{n2 k2} from the pairs
  double2 X = make_double2(0.0, 0.0);
#if DBX_WROW33_SPLIT && DBX_TW1T
  {
    // X[k2] = A + (-i) B and X[31 - k2] = A - (-i) B share A (cosine sums of the
    // folded sums) and B (sine sums of the folded differences): lane k2 <= 15
    // forms A, lane 31 - k2 forms B (real weights, tables.cpp), one exchange
    const bool isB = lane >= 16;
    const double sgn = isB ? -1.0 : 1.0;
    const double* __restrict__ wr = reinterpret_cast<const double*>(tw) + 2 * 32 * 48 + lane;
    const double2 y0 = buf[wslot(992)];
    double2 acc = isB ? make_double2(0.0, 0.0) : y0;
#pragma unroll
    for (int j = 1; j <= 15; ++j) {
      const double2 yj = buf[wslot(992 + j)], ym = buf[wslot(992 + 31 - j)];
      const double w = __ldg(wr + 32 * (j - 1));
      acc.x = fma(w, fma(sgn, ym.x, yj.x), acc.x);
      acc.y = fma(w, fma(sgn, ym.y, yj.y), acc.y);
    }
    const double2 P = make_double2(__shfl_sync(0xffffffffu, acc.x, 31 - lane), __shfl_sync(0xffffffffu, acc.y, 31 - lane));
    // A-lane: A + (B.y, -B.x) with B = P;  B-lane: A - (B.y, -B.x) with A = P, B = acc
    X = isB ? make_double2(P.x - acc.y, P.y + acc.x) : make_double2(acc.x + P.y, acc.y - P.x);
  }
#else
  {
    const double2 y0 = buf[wslot(992)];
    double2 A = y0, B = make_double2(0.0, 0.0);
    int e = 0;
#pragma unroll
    for (int j = 1; j <= 15; ++j) {
      e += lane;
      e = e >= 31 ? e - 31 : e;  // (j * lane) mod 31
      const double2 yj = buf[wslot(992 + j)], ym = buf[wslot(992 + 31 - j)];
#if DBX_TW1T
      const double2 w = __ldg(tw + 32 * (33 + j - 1) + lane);  // tw1t rows 33..47: W_31^{j lane}
#else
      const double2 w = __ldg(tw + 33 * e);  // (cos, -sin)(2 pi e / 31)
#endif
      const double2 a = cadd(yj, ym), b = csub(yj, ym);
      A.x = fma(w.x, a.x, A.x);
      A.y = fma(w.x, a.y, A.y);
      B.x = fma(-w.y, b.x, B.x);
      B.y = fma(-w.y, b.y, B.y);
    }
    X = cadd(A, fft::mul_si<S>(B));
  }
#endif
  __syncwarp();
  if (lane < 31) buf[wslot(992 + lane)] = X;
  __syncwarp();
}

// DFT_1023 whose level-1 inputs are already in registers (v[n1] = z at slot
// 31 n1 + lane): skips the fill's store pass and level 1's load pass.
__device__ __forceinline__ void wdft1023_pre(double2* buf, const double2* __restrict__ tw, int lane, double2* v) {
  if (lane < 31) level1_row(buf, tw, lane, v);
  __syncwarp();
  wdft1023_tail(buf, tw, lane);
}

// Packed-DST fill in level-1 geometry (DBX_WPRE): lane L holds the raw pair
// y_m = (line a, line b) at m = 31 n1 + L in v[n1], n1 < 33 (lane 31 shadows
// lane 0's column one row down, m = 31 (n1 + 1)), so the mirror y_{N-m} of
// every m sits in lane 31 - L at row 32 - n1: one shuffle per element instead
// of a line pass through shared memory.  In place:
//   z_m = s_m (y_m + y_{N-m} - S) + (y_m - y_{N-m} - D (1 - 2 m / N)) / 2
// (pk_fill's sd(j) for both halves: s and the sum are even in m <-> N - m, the
// difference and the ramp odd); S = D = 0 without the AR ramp.  z_0 = 0.
__device__ __forceinline__ double2 wshfl2(double2 x, int src) {
  return make_double2(__shfl_sync(0xffffffffu, x.x, src), __shfl_sync(0xffffffffu, x.y, src));
}
__device__ __forceinline__ double2 wfill_z(double2 y, double2 ym, double s, double r, double2 S, double2 D) {
  const double Aa = y.x + ym.x - S.x, Ba = (y.x - ym.x) - D.x * r;
  const double Ab = y.y + ym.y - S.y, Bb = (y.y - ym.y) - D.y * r;
  return make_double2(fma(s, Aa, 0.5 * Ba), fma(s, Ab, 0.5 * Bb));
}
__device__ __forceinline__ void wfill_pre(double2* v, const double* __restrict__ sn, int lane, double2 S, double2 D,
                                          double ri) {
  const int src = 31 - lane;
  const int ml = lane < 31 ? lane : 30;  // lane 31's outputs are unused: keep its table reads in range
#pragma unroll
  for (int n1 = 0; n1 <= 16; ++n1) {
    const int n1m = 32 - n1;
    const int m0 = 31 * n1 + ml, m1 = 31 * n1m + ml;
    const double s0 = __ldg(sn + m0), s1 = __ldg(sn + m1);
    const double2 t0 = wshfl2(v[n1m], src);  // y_{N - m0}
    const double2 t1 = n1 == n1m ? t0 : wshfl2(v[n1], src);  // y_{N - m1}
    const double2 z0 = wfill_z(v[n1], t0, s0, fma(-2.0 * ri, (double)m0, 1.0), S, D);
    const double2 z1 = wfill_z(v[n1m], t1, s1, fma(-2.0 * ri, (double)m1, 1.0), S, D);
    v[n1] = (n1 == 0 && lane == 0) ? make_double2(0.0, 0.0) : z0;
    if (n1 != n1m) v[n1m] = z1;
  }
}

// ---------------------------------------------------------------------------
// Component-split DFT_1023 (opt-in DBX_WDST_RI): each row DFT runs on a LANE PAIR,
// lane 2r holding the real and lane 2r+1 the imaginary component of every
// value of row r.  Real linear maps act on each component alone; the only
// re/im mixing — multiplication by S i (the sine half of a symmetric-pair DFT,
// the DFT-3's u) and the twiddle product — takes one __shfl_xor with the
// partner.  Both lanes run the same instructions on different data, so a
// lane holds 31-33 doubles of a row instead of 62-66 complex halves: the
// kernel fits 168 registers (3 CTAs = 12 warps per SM, the shared-memory cap)
// without spills.  16 rows per warp pass: level 1 in two passes (31 rows),
// level 2 in two passes (rows 0..31) + the cooperative row 32.
struct Ri {
  int h;            // 0: real lane, 1: imaginary lane
  double sgn_si;    // S i v on this lane's component = sgn_si * partner (S = -1)
  double sgn_mul;   // (v w).comp = own w.x + sgn_mul * partner w.y
};
__device__ __forceinline__ double partner(double v) { return __shfl_xor_sync(0xffffffffu, v, 1); }
// comp of S i v (S = -1: -i v = (v.y, -v.x))
__device__ __forceinline__ double si_comp(const Ri& R, double v) { return R.sgn_si * partner(v); }

__device__ __forceinline__ void level1_row_ri(double* bd, const double2* __restrict__ tw, int n2, bool act,
                                              const Ri& R, double* v) {
  constexpr double c3 = 0.86602540378443864676372317075293618;  // sqrt(3)/2
#pragma unroll
  for (int b = 0; b < 11; ++b) {
    const int i0 = (3 * b) % 33, i1 = (11 + 3 * b) % 33, i2 = (22 + 3 * b) % 33;
    const double t = v[i1] + v[i2];
    const double u = si_comp(R, c3 * (v[i1] - v[i2]));
    const double m = v[i0] - 0.5 * t;
    v[i0] = v[i0] + t;
    v[i1] = m + u;
    v[i2] = m - u;
  }
  auto put = [&](int k1, double x) {
    if (k1 != 0) {
      const double2 w = __ldg(tw + n2 * k1);  // n2 k1 <= 990
      x = fma(x, w.x, R.sgn_mul * partner(x) * w.y);
    }
    if (act) bd[2 * (31 * k1 + n2) + R.h] = x;
  };
#pragma unroll
  for (int ka = 0; ka < 3; ++ka) {
    double* u[11];
#pragma unroll
    for (int b = 0; b < 11; ++b) u[b] = &v[(11 * ka + 3 * b) % 33];
    const double x0 = *u[0];
    double sum = x0;
#pragma unroll
    for (int j = 1; j <= 5; ++j) {
      const double pp = *u[j] + *u[11 - j], mm = *u[j] - *u[11 - j];
      *u[j] = pp;
      *u[11 - j] = mm;
      sum += pp;
    }
    put((22 * ka) % 33, sum);
#pragma unroll
    for (int k = 1; k <= 5; ++k) {
      double A = x0, B = 0.0;
#pragma unroll
      for (int j = 1; j <= 5; ++j) {
        const int e = (j * k) % 11;
        A = fma(ccs<11>(e), *u[j], A);
        B = fma(scs<11>(e), *u[11 - j], B);
      }
      const double sb = si_comp(R, B);
      put((22 * ka + 12 * k) % 33, A + sb);
      put((22 * ka + 12 * (11 - k)) % 33, A - sb);
    }
  }
}

__device__ __forceinline__ void wdft1023_ri(double2* buf, const double2* __restrict__ tw, int lane) {
  Ri R;
  R.h = lane & 1;
  R.sgn_si = R.h ? -1.0 : 1.0;
  R.sgn_mul = R.h ? 1.0 : -1.0;
  double* bd = reinterpret_cast<double*>(buf);
  const int r = lane >> 1;
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    const int n2 = 16 * pass + r;
    const bool act = n2 < 31;
    const int nr = act ? n2 : 30;  // lanes without a row shadow row 30 (shuffle partners, no stores)
    double v[33];
#pragma unroll
    for (int n1 = 0; n1 < 33; ++n1) v[n1] = bd[2 * (31 * n1 + nr) + R.h];
    level1_row_ri(bd, tw, nr, act, R, v);
  }
  __syncwarp();
#pragma unroll 1
  for (int pass = 0; pass < 2; ++pass) {
    const int base = 31 * (16 * pass + r);
    double v[31];
#pragma unroll
    for (int j = 0; j < 31; ++j) v[j] = bd[2 * (base + j) + R.h];
    const double x0 = v[0];
    double sum = x0;
#pragma unroll
    for (int j = 1; j <= 15; ++j) {
      const double a = v[j] + v[31 - j], b = v[j] - v[31 - j];
      v[j] = a;
      v[31 - j] = b;
      sum += a;
    }
    bd[2 * base + R.h] = sum;
#pragma unroll
    for (int k = 1; k <= 15; ++k) {
      double A = x0, B = 0.0;
#pragma unroll
      for (int j = 1; j <= 15; ++j) {
        const int e = (j * k) % 31;
        A = fma(ccs<31>(e), v[j], A);
        B = fma(scs<31>(e), v[31 - j], B);
      }
      const double sb = si_comp(R, B);
      bd[2 * (base + k) + R.h] = A + sb;
      bd[2 * (base + 31 - k) + R.h] = A - sb;
    }
  }
  // row k1 = 32: one complex output per lane (as in wdft1023)
  double2 X = make_double2(0.0, 0.0);
  {
    constexpr int S = -1;
    const double2 y0 = buf[992];
    double2 A = y0, B = make_double2(0.0, 0.0);
    int e = 0;
#pragma unroll
    for (int j = 1; j <= 15; ++j) {
      e += lane;
      e = e >= 31 ? e - 31 : e;
      const double2 yj = buf[992 + j], ym = buf[992 + 31 - j];
      const double2 w = __ldg(tw + 33 * e);
      const double2 a = cadd(yj, ym), b = csub(yj, ym);
      A.x = fma(w.x, a.x, A.x);
      A.y = fma(w.x, a.y, A.y);
      B.x = fma(-w.y, b.x, B.x);
      B.y = fma(-w.y, b.y, B.y);
    }
    X = cadd(A, fft::mul_si<S>(B));
  }
  __syncwarp();
  if (lane < 31) buf[992 + lane] = X;
  __syncwarp();
}

// Split + odd scan in place: the DFT outputs Y_l (slot wpos(l)) become the
// two real output lines, out[k] = (X^a_k, X^b_k) at slot(k), k in [0, 1024),
// in the scaled DST-I convention of pk_split2 + odd_scans2.  Lane L owns the
// pairs l in [16L, 16L+16) (outputs k in [32L, 32L+32)): all its Y reads
// precede a __syncwarp, then its outputs overwrite the line.
__device__ __forceinline__ void wsplit(double2* buf, int lane, double hs, double sc) {
  double2 zl[16], zm[16];
  double ta = 0.0, tb = 0.0;
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int l = 16 * lane + i;
    zl[i] = buf[wpos(l)];
    zm[i] = buf[wpos(l == 0 ? 0 : kWN - l)];
  }
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int l = 16 * lane + i;
    if (2 * l + 1 <= kWN - 1) {
      const double f = l == 0 ? 0.25 : 0.5;
      ta += f * (zl[i].x + zm[i].x);
      tb += f * (zl[i].y + zm[i].y);
    }
  }
  double ia = ta, ib = tb;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double ya = __shfl_up_sync(0xffffffffu, ia, d), yb = __shfl_up_sync(0xffffffffu, ib, d);
    if (lane >= d) {
      ia += ya;
      ib += yb;
    }
  }
  double pa = ia - ta, pb = ib - tb;  // exclusive offsets; then the lane's own running sums
  __syncwarp();  // every lane's Y reads precede the outputs (other layout, same slots)
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    const int l = 16 * lane + i;
    const double ea = l >= 1 ? hs * (zm[i].y - zl[i].y) : 0.0;
    const double eb = l >= 1 ? hs * (zl[i].x - zm[i].x) : 0.0;
    if (2 * l + 1 <= kWN - 1) {
      const double f = l == 0 ? 0.25 : 0.5;
      pa += f * (zl[i].x + zm[i].x);
      pb += f * (zl[i].y + zm[i].y);
    }
    buf[oslot(2 * l)] = make_double2(ea, eb);
    buf[oslot(2 * l + 1)] = make_double2(pa * sc, pb * sc);
  }
  __syncwarp();
}

#if DBX_WDST_RI
#define WDFT wdft1023_ri
#else
#define WDFT wdft1023
#endif

// ---------------------------------------------------------------------------
// DFT_255 (C1's 256-point lines, N = 255 = 17 * 15) in the same warp-owned
// form: level 1, lane n2 < 17: x[17 n1 + n2], n1 < 15 -> in-register DFT-15
// (3 x 5 prime factor) -> * W_255^{n2 k1} -> slot 17 k1 + n2; level 2, lane
// k1 < 15: the 17 contiguous slots 17 k1 + n2 -> DFT-17 (symmetric pairs) ->
// X[k1 + 15 k2] at slot 17 k1 + k2.
__device__ __forceinline__ int oslot255(int k) { return k ^ ((k >> 3) & 7); }
__device__ __forceinline__ int wpos255(int l) {
  const int k2 = l / 15;
  return 17 * (l - 15 * k2) + k2;
}

__device__ __forceinline__ void wdft255(double2* buf, const double2* __restrict__ tw, int lane) {
  constexpr int S = -1;
  if (lane < 17) {
    double2 v[15];
#pragma unroll
    for (int n1 = 0; n1 < 15; ++n1) v[n1] = buf[17 * n1 + lane];
    fft::dft15<S>(v);
#pragma unroll
    for (int k1 = 0; k1 < 15; ++k1) {
      double2 x = v[k1];
#if DBX_TW1T
      if (k1 != 0) x = fft::cmul(x, __ldg(tw + 32 * k1 + lane));  // tw1t [k1][lane]
#else
      if (k1 != 0) x = fft::cmul(x, __ldg(tw + lane * k1));  // n2 k1 <= 224
#endif
      buf[17 * k1 + lane] = x;
    }
  }
  __syncwarp();
  if (lane < 15) {
    const int base = 17 * lane;
    double2 v[17];
#pragma unroll
    for (int j = 0; j < 17; ++j) v[j] = buf[base + j];
    const double2 x0 = v[0];
    double2 sum = x0;
#pragma unroll
    for (int j = 1; j <= 8; ++j) {
      const double2 a = cadd(v[j], v[17 - j]), b = csub(v[j], v[17 - j]);
      v[j] = a;
      v[17 - j] = b;
      sum = cadd(sum, a);
    }
    buf[base] = sum;
#pragma unroll
    for (int k = 1; k <= 8; ++k) {
      double2 A = x0, B = make_double2(0.0, 0.0);
#pragma unroll
      for (int j = 1; j <= 8; ++j) {
        const int e = (j * k) % 17;
        A.x = fma(ccs<17>(e), v[j].x, A.x);
        A.y = fma(ccs<17>(e), v[j].y, A.y);
        B.x = fma(scs<17>(e), v[17 - j].x, B.x);
        B.y = fma(scs<17>(e), v[17 - j].y, B.y);
      }
      const double2 sb = fft::mul_si<S>(B);
      buf[base + k] = cadd(A, sb);
      buf[base + 17 - k] = csub(A, sb);
    }
  }
  __syncwarp();
}

// wsplit for N = 255: lane L owns the pairs l in [4L, 4L+4) (outputs
// k in [8L, 8L+8)); same convention as wsplit.
__device__ __forceinline__ void wsplit255(double2* buf, int lane, double hs, double sc) {
  constexpr int NN = 255;
  double2 zl[4], zm[4];
  double ta = 0.0, tb = 0.0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int l = 4 * lane + i;
    zl[i] = buf[wpos255(l)];
    zm[i] = buf[wpos255(l == 0 ? 0 : NN - l)];
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int l = 4 * lane + i;
    if (2 * l + 1 <= NN - 1) {
      const double f = l == 0 ? 0.25 : 0.5;
      ta += f * (zl[i].x + zm[i].x);
      tb += f * (zl[i].y + zm[i].y);
    }
  }
  double ia = ta, ib = tb;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double ya = __shfl_up_sync(0xffffffffu, ia, d), yb = __shfl_up_sync(0xffffffffu, ib, d);
    if (lane >= d) {
      ia += ya;
      ib += yb;
    }
  }
  double pa = ia - ta, pb = ib - tb;
  __syncwarp();
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int l = 4 * lane + i;
    const double ea = l >= 1 ? hs * (zm[i].y - zl[i].y) : 0.0;
    const double eb = l >= 1 ? hs * (zl[i].x - zm[i].x) : 0.0;
    if (2 * l + 1 <= NN - 1) {
      const double f = l == 0 ? 0.25 : 0.5;
      pa += f * (zl[i].x + zm[i].x);
      pb += f * (zl[i].y + zm[i].y);
    }
    buf[oslot255(2 * l)] = make_double2(ea, eb);
    buf[oslot255(2 * l + 1)] = make_double2(pa * sc, pb * sc);
  }
  __syncwarp();
}

// Geometry traits of the warp-owned kernels: DFT length N (line n = N + 1),
// fill rows J = (N/2 + 1) / 32 and outputs K = n / 32 per lane, warps per CTA,
// per-warp line stride (+1 slot: conflict-free cross-warp reads) and the x-row
// stride RLS of rows_t_axpy_w (= 4 mod 16 for sep_row_stencil_T, room for the
// 16-slot front offset and a q2 <= 15 extension).
struct W1023 {
  static constexpr int N = 1023, LINE = 1024, J = 16, K = 32, WARPS = kWWarps;
  static constexpr int STRIDE = LINE + DBX_WSTRIDE_PAD, RLS = 1076;
  __device__ static int oslot(int k) { return ::dbx::oslot(k); }
  static constexpr bool PRE = DBX_WPRE && DBX_TW1T && !DBX_WDST_RI;
  __device__ static void dft(double2* buf, const BlueTables& bt, int lane) {
    WDFT(buf, (DBX_TW1T && !DBX_WDST_RI) ? bt.tw1t : bt.tw, lane);
  }
  __device__ static void dft_pre(double2* buf, const BlueTables& bt, int lane, double2* v) {
    wdft1023_pre(buf, bt.tw1t, lane, v);
  }
  __device__ static void split(double2* buf, int lane, double hs, double sc) { wsplit(buf, lane, hs, sc); }
};
#ifndef DBX_W255_WARPS
#define DBX_W255_WARPS 2  // 64 CTAs for a 256^2 image (A/B: 2018 vs 1968 Mpx-it/s at 4)
#endif
struct W255 {
  static constexpr int N = 255, LINE = 256, J = 4, K = 8, WARPS = DBX_W255_WARPS;
  static constexpr int STRIDE = LINE + DBX_WSTRIDE_PAD, RLS = 308;
  __device__ static int oslot(int k) { return oslot255(k); }
  static constexpr bool PRE = false;
  __device__ static void dft(double2* buf, const BlueTables& bt, int lane) {
    wdft255(buf, DBX_TW1T ? bt.tw1t : bt.tw, lane);
  }
  __device__ static void dft_pre(double2*, const BlueTables&, int, double2*) {}
  __device__ static void split(double2* buf, int lane, double hs, double sc) { wsplit255(buf, lane, hs, sc); }
};

// CTA_STORE (n2 a multiple of 2 W::WARPS): after one CTA barrier the 4 warps'
// outputs leave as 64-byte row segments (8 columns) instead of each warp's
// 16-byte pieces at 32 different rows per store instruction.
template <class W, bool CTA_STORE>
__global__ void __launch_bounds__(32 * W::WARPS, DBX_WDST_MINB) dst_tcols_w(SpecArgs a) {
  DBX_PDL_WAIT();
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 wsm[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2* buf = wsm + (size_t)w * W::STRIDE;
  const BlueTables& bt = a.blue1;
  const int n = a.n1, n2 = a.n2;
  const size_t N = (size_t)n * n2;
  const int c = 2 * (W::WARPS * blockIdx.x + w);  // columns c, c+1
  if (c >= n2) return;                           // warp-uniform; no CTA barriers below
  const bool hb = c + 1 < n2;
  const double ri = bt.rinv, hs = 0.5 * bt.scale, sc = bt.scale;
  const double* __restrict__ sn = bt.sn;
  // ---- T~ (ar_inverse, transforms.hpp:163-173) of columns c, c+1 (contiguous
  // in u^T): lane L fills the mirror pairs p = L + 32 j <= N/2 and N - p
#if DBX_WDST_PREFETCH > 0
  if (lane == 0) {
    const long cta = (long)b * gridDim.x + blockIdx.x + (long)DBX_WDST_PREFETCH * 148 * DBX_WDST_MINB;
    const long pb = cta / gridDim.x, pc = 2 * (W::WARPS * (cta - pb * gridDim.x) + w);
    if (pb < a.batch && pc + 1 < n2) prefetch_l2(a.in + (size_t)pb * N + (size_t)pc * n, (unsigned)(2 * n * 8));
  }
#endif
  const double* ua = a.in + (size_t)b * N + (size_t)c * n;
  const double* ub = hb ? ua + n : ua;
  const double x0a = __ldg(ua), xea = __ldg(ua + n - 1), x0b = __ldg(ub), xeb = __ldg(ub + n - 1);
  const double sa = x0a + xea, sb = x0b + xeb, da = x0a - xea, db = x0b - xeb;
  if constexpr (W::PRE) {
    // level-1 geometry: lane's column m = 31 n1 + lane of both lines (wfill_pre)
    double2 v[33];
#pragma unroll
    for (int n1 = 0; n1 < 33; ++n1)
      v[n1] = make_double2(__ldg(ua + 31 * n1 + lane), hb ? __ldg(ub + 31 * n1 + lane) : 0.0);
    wfill_pre(v, sn, lane, make_double2(sa, hb ? sb : 0.0), make_double2(da, hb ? db : 0.0), ri);
    W::dft_pre(buf, bt, lane, v);
  } else {
    // every global load of the fill in flight at once (one HBM latency per
    // item instead of one per unrolled group)
    double ap[W::J], aq[W::J], bp[W::J], bq[W::J];
  #pragma unroll
    for (int j = 0; j < W::J; ++j) {
      const int p = lane + 32 * j, q = W::N - p;  // p in [0, 511], q in [512, 1023]
      ap[j] = __ldg(ua + p);
      aq[j] = __ldg(ua + q);
      bp[j] = __ldg(ub + p);
      bq[j] = __ldg(ub + q);
    }
  #pragma unroll
    for (int j = 0; j < W::J; ++j) {
      const int p = lane + 32 * j, q = W::N - p;
      const double r = fma(-2.0 * ri, (double)p, 1.0), s = __ldg(sn + p);
      const double Aa = ap[j] + aq[j] - sa, Ba = (ap[j] - aq[j]) - da * r;  // sd(j) of pk_fill
      const double Ab = bp[j] + bq[j] - sb, Bb = (bp[j] - bq[j]) - db * r;
      if (p == 0) {
        buf[wslot(0)] = make_double2(0.0, 0.0);
      } else {
        buf[wslot(p)] = make_double2(fma(s, Aa, 0.5 * Ba), hb ? fma(s, Ab, 0.5 * Bb) : 0.0);
        buf[wslot(q)] = make_double2(fma(s, Aa, -0.5 * Ba), hb ? fma(s, Ab, -0.5 * Bb) : 0.0);
      }
    }
  __syncwarp();
    W::dft(buf, bt, lane);
  }
  W::split(buf, lane, hs, sc);
  // ---- v = u o d (d^T rows c, c+1: L2-resident, shared by the batch), then
  // the T fill from the same mirror pairs (reads and writes slots p, N - p only)
  const double* dA = a.dT + (size_t)b * a.dstride + (size_t)c * n;
  const double* dB = hb ? dA + n : dA;
  const double a0a = x0a * __ldg(dA), a1a = xea * __ldg(dA + n - 1);
  const double a0b = x0b * __ldg(dB), a1b = xeb * __ldg(dB + n - 1);
  if constexpr (W::PRE) {
    // y = out o d in level-1 geometry (column m = 31 n1 + lane), mirrors by shuffle
    double2 v[33];
#pragma unroll
    for (int n1 = 0; n1 < 33; ++n1) {
      const int m = 31 * n1 + lane;
      const double2 o = buf[W::oslot(m)];
      v[n1] = make_double2(o.x * __ldg(dA + m), o.y * __ldg(dB + m));
    }
    __syncwarp();  // every read of the split outputs precedes level 1's stores
    wfill_pre(v, sn, lane, make_double2(0.0, 0.0), make_double2(0.0, 0.0), ri);
    W::dft_pre(buf, bt, lane, v);
  } else {
    // d loads all in flight first; then per mirror row j: read out[p], out[q]
    // (oslot), syncwarp, write z_p, z_q (slot p, q).  Every slot a lane writes
    // in row j aliases only reads of the same row j (oslot permutes within
    // 8-aligned groups keyed by k >> 5), so one __syncwarp per row orders them.
    double dpa[W::J], dqa[W::J], dpb[W::J], dqb[W::J];
  #pragma unroll
    for (int j = 0; j < W::J; ++j) {
      const int p = lane + 32 * j, q = W::N - p;
      dpa[j] = __ldg(dA + p);
      dqa[j] = __ldg(dA + q);
      dpb[j] = __ldg(dB + p);
      dqb[j] = __ldg(dB + q);
    }
  #pragma unroll
    for (int j = 0; j < W::J; ++j) {
      const int p = lane + 32 * j, q = W::N - p;  // p = 0: z_0 = 0 (q = 1023 is no DFT slot)
      const double2 op = buf[W::oslot(p)], oq = buf[W::oslot(q)];
      const double mpa = op.x * dpa[j], mqa = oq.x * dqa[j];
      const double mpb = op.y * dpb[j], mqb = oq.y * dqb[j];
      const double s = __ldg(sn + p);
      const double Aa = mpa + mqa, Ba = mpa - mqa, Ab = mpb + mqb, Bb = mpb - mqb;
      __syncwarp();
      if (p == 0) {
        buf[wslot(0)] = make_double2(0.0, 0.0);
      } else {
        buf[wslot(p)] = make_double2(fma(s, Aa, 0.5 * Ba), fma(s, Ab, 0.5 * Bb));
        buf[wslot(q)] = make_double2(fma(s, Aa, -0.5 * Ba), fma(s, Ab, -0.5 * Bb));
      }
    }
  __syncwarp();
    W::dft(buf, bt, lane);
  }
  W::split(buf, lane, hs, sc);
  // ---- T (ar_forward, transforms.hpp:148-160): w_0 = a0, w_{n-1} = a1,
  // interior DST + ramp a0 (1 - k/(n-1)) + a1 k/(n-1); row-major stores
  if constexpr (CTA_STORE) {
    __shared__ double2 ramp[W::WARPS][2];
    if (lane == 0) {
      ramp[w][0] = make_double2(a0a, a0b);
      ramp[w][1] = make_double2(a1a, a1b);
    }
    __syncthreads();
    double* outb = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N)) +
                   2 * W::WARPS * blockIdx.x;
#pragma unroll 4
    for (int idx = threadIdx.x; idx < W::WARPS * n; idx += 32 * W::WARPS) {
      const int ww = idx & (W::WARPS - 1), k = idx / W::WARPS;
      const double2 o = wsm[(size_t)ww * W::STRIDE + W::oslot(k)];
      const double2 r0v = ramp[ww][0], r1v = ramp[ww][1];
      const double t1 = (double)k * ri;
      double wa = o.x + r0v.x * (1.0 - t1) + r1v.x * t1;
      double wb = o.y + r0v.y * (1.0 - t1) + r1v.y * t1;
      if (k == 0) { wa = r0v.x; wb = r0v.y; }
      if (k == n - 1) { wa = r1v.x; wb = r1v.y; }
      *reinterpret_cast<double2*>(outb + (size_t)k * n2 + 2 * ww) = make_double2(wa, wb);
    }
    return;
  }
  double* out = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N)) + c;
#pragma unroll 8
  for (int j = 0; j < W::K; ++j) {
    const int k = lane + 32 * j;
    const double2 o = buf[W::oslot(k)];
    const double t1 = (double)k * ri;
    double wa = o.x + a0a * (1.0 - t1) + a1a * t1;
    double wb = o.y + a0b * (1.0 - t1) + a1b * t1;
    if (k == 0) { wa = a0a; wb = a0b; }
    if (k == n - 1) { wa = a1a; wb = a1b; }
    if (hb) *reinterpret_cast<double2*>(out + (size_t)k * n2) = make_double2(wa, wb);
    else out[(size_t)k * n2] = wa;
  }
}


// ---------------------------------------------------------------------------
// Warp-owned ROW kernels of the separable fused pipeline for n2 = 1024 (the
// rows of C3): the same DFT_1023 / split as dst_tcols_w, one warp per packed
// row pair, and ONE CTA barrier before the cooperative transposed stores.
// CTA = W::WARPS warps = 8 rows r0 .. r0+7.
//
// rows_tt_w (K2, replaces rows_ainv_tt<SEP>): s = A'r rows (row-major, ybuf)
// -> T~ along the rows (ar_inverse, transforms.hpp:163-173) -> u^T[k][row]
// (64-byte row segments: 8 rows per column k).

template <class W>
__global__ void __launch_bounds__(32 * W::WARPS, DBX_WDST_MINB) rows_tt_w(SpecArgs a) {
  DBX_PDL_WAIT();
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 wsm[];
  __shared__ double ends[2 * W::WARPS][2];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2* buf = wsm + (size_t)w * W::STRIDE;
  const BlueTables& bt = a.blue2;
  const int n1 = a.n1, n2 = a.n2;
  const size_t N = (size_t)n1 * n2;
  const int r0 = 2 * W::WARPS * blockIdx.x, r = r0 + 2 * w;  // rows r, r+1
  const bool act = r < n1, hb = r + 1 < n1;
  if (act) {
    const double ri = bt.rinv, hs = 0.5 * bt.scale, sc = bt.scale;
    const double* __restrict__ sn = bt.sn;
    const double* ua = reinterpret_cast<const double*>(a.ybuf) + (size_t)b * N + (size_t)r * n2;
    const double* ub = hb ? ua + n2 : ua;
    const double x0a = __ldg(ua), xea = __ldg(ua + n2 - 1), x0b = __ldg(ub), xeb = __ldg(ub + n2 - 1);
    if (lane == 0) {
      ends[2 * w][0] = x0a; ends[2 * w][1] = xea;
      ends[2 * w + 1][0] = x0b; ends[2 * w + 1][1] = xeb;
    }
    const double sa = x0a + xea, sb = x0b + xeb, da = x0a - xea, db = x0b - xeb;
    if constexpr (W::PRE) {
      double2 v[33];
#pragma unroll
      for (int n1 = 0; n1 < 33; ++n1)
        v[n1] = make_double2(__ldg(ua + 31 * n1 + lane), hb ? __ldg(ub + 31 * n1 + lane) : 0.0);
      wfill_pre(v, sn, lane, make_double2(sa, hb ? sb : 0.0), make_double2(da, hb ? db : 0.0), ri);
      W::dft_pre(buf, bt, lane, v);
    } else {
      double ap[W::J], aq[W::J], bp[W::J], bq[W::J];
  #pragma unroll
      for (int j = 0; j < W::J; ++j) {
        const int p = lane + 32 * j, q = W::N - p;
        ap[j] = __ldg(ua + p);
        aq[j] = __ldg(ua + q);
        bp[j] = __ldg(ub + p);
        bq[j] = __ldg(ub + q);
      }
  #pragma unroll
      for (int j = 0; j < W::J; ++j) {
        const int p = lane + 32 * j, q = W::N - p;
        const double rr = fma(-2.0 * ri, (double)p, 1.0), s = __ldg(sn + p);
        const double Aa = ap[j] + aq[j] - sa, Ba = (ap[j] - aq[j]) - da * rr;
        const double Ab = bp[j] + bq[j] - sb, Bb = (bp[j] - bq[j]) - db * rr;
        if (p == 0) {
          buf[wslot(0)] = make_double2(0.0, 0.0);
        } else {
          buf[wslot(p)] = make_double2(fma(s, Aa, 0.5 * Ba), hb ? fma(s, Ab, 0.5 * Bb) : 0.0);
          buf[wslot(q)] = make_double2(fma(s, Aa, -0.5 * Ba), hb ? fma(s, Ab, -0.5 * Bb) : 0.0);
        }
      }
    __syncwarp();
      W::dft(buf, bt, lane);
    }
    W::split(buf, lane, hs, sc);
  }
  __syncthreads();
  // u^T[k][r0 + 2 ww .. + 1] from warp ww's line: 4 x 16 bytes per column k
  double* uT = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N));
  const double al = bt.alpha;
#pragma unroll 4
  for (int idx = threadIdx.x; idx < W::WARPS * n2; idx += 32 * W::WARPS) {
    const int ww = idx & (W::WARPS - 1), k = idx / W::WARPS;
    const int rr = r0 + 2 * ww;
    if (rr >= n1) continue;
    double2 o = wsm[(size_t)ww * W::STRIDE + W::oslot(k)];
    if (k == 0) o = make_double2(al * ends[2 * ww][0], al * ends[2 * ww + 1][0]);
    if (k == n2 - 1) o = make_double2(al * ends[2 * ww][1], al * ends[2 * ww + 1][1]);
    double* dst = uT + (size_t)k * n1 + rr;
    if (rr + 1 < n1) *reinterpret_cast<double2*>(dst) = o;
    else *dst = o.x;
  }
}

// rows_t_axpy_w (K4, replaces rows_t_axpy_afwd<SEP>): T along the rows of v
// (ar_forward, transforms.hpp:148-160) -> x_k = x_{k-1} + tau T v
// (solver.hpp:106) with ||x||^2, ||x - f||^2 partials -> the x_k rows,
// AR-extended in place (boundary.hpp:56-62), correlated with A's row taps into
// Z^T (sep_row_stencil_T, 4 rows at a time).  Warp w's region (W::RLS
// double2) holds its DFT line, then its two x rows at double offsets 16 and
// W::RLS + 16 of the CTA's 8-row stencil block.
template <class W>
__global__ void __launch_bounds__(32 * W::WARPS, DBX_WDST_MINB) rows_t_axpy_w(SpecArgs a) {
  DBX_PDL_WAIT();
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 wsm[];
  __shared__ double red[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  double2* buf = wsm + (size_t)w * W::RLS;
  double* xs = reinterpret_cast<double*>(wsm);  // 8 rows at stride W::RLS, data at offset 16
  const BlueTables& bt = a.blue2;
  const int n1 = a.n1, n2 = a.n2, q2 = a.q2;
  const size_t N = (size_t)n1 * n2;
  const int r0 = 2 * W::WARPS * blockIdx.x, r = r0 + 2 * w;
  const bool act = r < n1, hb = r + 1 < n1;
  const double* xo = resolve_ptr(a.xold, a.st, a.xoldsel, b, a.batch, N) + (size_t)r * n2;
  const double* fimg = a.f ? a.f + (size_t)b * N + (size_t)r * n2 : nullptr;
  // x_{k-1} and f rows are read after the two DFTs: start them towards L2 now
  if (act && lane == 0) {
    prefetch_l2(xo, (unsigned)((hb ? 2 : 1) * n2 * 8));
    if (fimg) prefetch_l2(fimg, (unsigned)((hb ? 2 : 1) * n2 * 8));
  }
  double p0 = 0.0, p1 = 0.0;
  if (act) {
    const double ri = bt.rinv, hs = 0.5 * bt.scale, sc = bt.scale, tau = a.tau, ia = 1.0 / bt.alpha;
    const double* __restrict__ sn = bt.sn;
    const double* va = a.in + (size_t)b * N + (size_t)r * n2;
    const double* vb = hb ? va + n2 : va;
    const double a0a = ia * __ldg(va), a1a = ia * __ldg(va + n2 - 1);
    const double a0b = ia * __ldg(vb), a1b = ia * __ldg(vb + n2 - 1);
    if constexpr (W::PRE) {
      double2 v[33];
#pragma unroll
      for (int n1 = 0; n1 < 33; ++n1)
        v[n1] = make_double2(__ldg(va + 31 * n1 + lane), hb ? __ldg(vb + 31 * n1 + lane) : 0.0);
      wfill_pre(v, sn, lane, make_double2(0.0, 0.0), make_double2(0.0, 0.0), ri);
      W::dft_pre(buf, bt, lane, v);
    } else {
      double ap[W::J], aq[W::J], bp[W::J], bq[W::J];
  #pragma unroll
      for (int j = 0; j < W::J; ++j) {
        const int p = lane + 32 * j, q = W::N - p;
        ap[j] = __ldg(va + p);
        aq[j] = __ldg(va + q);
        bp[j] = __ldg(vb + p);
        bq[j] = __ldg(vb + q);
      }
  #pragma unroll
      for (int j = 0; j < W::J; ++j) {
        const int p = lane + 32 * j, q = W::N - p;
        const double s = __ldg(sn + p);
        const double Aa = ap[j] + aq[j], Ba = ap[j] - aq[j];
        const double Ab = bp[j] + bq[j], Bb = bp[j] - bq[j];
        if (p == 0) {
          buf[wslot(0)] = make_double2(0.0, 0.0);
        } else {
          buf[wslot(p)] = make_double2(fma(s, Aa, 0.5 * Ba), hb ? fma(s, Ab, 0.5 * Bb) : 0.0);
          buf[wslot(q)] = make_double2(fma(s, Aa, -0.5 * Ba), hb ? fma(s, Ab, -0.5 * Bb) : 0.0);
        }
      }
    __syncwarp();
      W::dft(buf, bt, lane);
    }
    W::split(buf, lane, hs, sc);
    // x_k = x_{k-1} + tau w, w = the T output with the ramp; all line reads
    // precede the x row writes into the same region
    double* xn = const_cast<double*>(resolve_ptr(a.out, a.st, a.outsel, b, a.batch, N)) + (size_t)r * n2;
    double2 ov[W::K];
#pragma unroll
    for (int j = 0; j < W::K; ++j) ov[j] = buf[W::oslot(lane + 32 * j)];
    __syncwarp();  // the x rows overwrite the line below
    double* ra = xs + (size_t)(2 * w) * W::RLS + 16;
    double* rb = ra + W::RLS;
    // x_{k-1} / f loads eight columns deep per lane (the x_k stores would
    // otherwise keep the compiler from hoisting them: one L2 round trip per
    // group instead of per element)
#pragma unroll
    for (int jc = 0; jc < W::K; jc += 8) {
      double oa[8], ob[8], fa[8], fb[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = lane + 32 * (jc + u);
        oa[u] = __ldcs(xo + k);
        ob[u] = hb ? __ldcs(xo + n2 + k) : 0.0;
        fa[u] = fimg ? __ldcs(fimg + k) : 0.0;
        fb[u] = (fimg && hb) ? __ldcs(fimg + n2 + k) : 0.0;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int k = lane + 32 * (jc + u);
        const double2 o = ov[jc + u];
        const double t1 = (double)k * ri;
        double wa = o.x + a0a * (1.0 - t1) + a1a * t1;
        double wb = o.y + a0b * (1.0 - t1) + a1b * t1;
        if (k == 0) { wa = a0a; wb = a0b; }
        if (k == n2 - 1) { wa = a1a; wb = a1b; }
        const double xa = oa[u] + tau * wa;
        xn[k] = xa;
        ra[k] = xa;
        p0 += xa * xa;
        if (fimg) {
          const double e = xa - fa[u];
          p1 += e * e;
        }
        double xb = 0.0;
        if (hb) {
          xb = ob[u] + tau * wb;
          xn[n2 + k] = xb;
          p0 += xb * xb;
          if (fimg) {
            const double e = xb - fb[u];
            p1 += e * e;
          }
        }
        rb[k] = xb;
      }
    }
    __syncwarp();
    // AR extension of both rows (f_{-k} = 2 f_0 - f_k, f_{n-1+k} = 2 f_{n-1} - f_{n-1-k})
    for (int m = lane; m < 2 * q2; m += 32) {
      if (m < q2) {
        const int k = q2 - m;
        ra[-k] = 2.0 * ra[0] - ra[k];
        rb[-k] = 2.0 * rb[0] - rb[k];
      } else {
        const int k = m - q2 + 1;
        ra[n2 - 1 + k] = 2.0 * ra[n2 - 1] - ra[n2 - 1 - k];
        rb[n2 - 1 + k] = 2.0 * rb[n2 - 1] - rb[n2 - 1 - k];
      }
    }
  }
  __syncthreads();
  double* zT = reinterpret_cast<double*>(a.zbuf) + (size_t)b * N + r0;
  for (int h0 = 0; h0 < 2 * W::WARPS; h0 += 4) {
    const int nl = n1 - r0 - h0 < 4 ? n1 - r0 - h0 : 4;
    if (nl > 0) sep_row_pass(xs + (size_t)h0 * W::RLS + 16 - q2, W::RLS, a.conv, q2, n2, nl, zT + h0, n1);
  }
  if (a.part.p) {
    double* P = a.part.p + (size_t)b * NUM_SLOTS * a.part.cap;
    const double s0 = block_sum<32 * W::WARPS>(p0, red);
    if (threadIdx.x == 0) P[SLOT_X2 * a.part.cap + blockIdx.x] = s0;
    const double s1 = block_sum<32 * W::WARPS>(p1, red);
    if (threadIdx.x == 0) P[SLOT_XF2 * a.part.cap + blockIdx.x] = s1;
  }
}

}  // namespace

// Warp-owned column half of D for 1024- and 256-point columns (direct 1023-
// and 255-point cores); returns the CTA count, or -1 when the shape is not
// this kernel's.
template <class W>
int launch_tcols_w_t(const SpecArgs& a, cudaStream_t s) {
  const size_t bytes = (size_t)W::WARPS * W::STRIDE * sizeof(double2);
  dim3 grid((a.n2 + 2 * W::WARPS - 1) / (2 * W::WARPS), a.batch);
  if (a.n2 % (2 * W::WARPS) == 0 && kWdstCtaStore) {
    static AttrOnce attr;
    if (!attr.ensure(dst_tcols_w<W, true>, bytes)) return -1;
    launch_k(dst_tcols_w<W, true>, grid, 32 * W::WARPS, bytes, s, a);
  } else {
    static AttrOnce attr;
    if (!attr.ensure(dst_tcols_w<W, false>, bytes)) return -1;
    launch_k(dst_tcols_w<W, false>, grid, 32 * W::WARPS, bytes, s, a);
  }
  return (int)grid.x;
}

int launch_dst_tcols_w(const SpecArgs& a, cudaStream_t s) {
  if (a.n1 == 1024 && a.blue1.N == W1023::N) return launch_tcols_w_t<W1023>(a, s);
  if (a.n1 == 256 && a.blue1.N == W255::N && kW255) return launch_tcols_w_t<W255>(a, s);
  return -1;
}

template <class W>
int launch_rows_w_t(int which, const SpecArgs& a, cudaStream_t s) {
  dim3 grid((a.n1 + 2 * W::WARPS - 1) / (2 * W::WARPS), a.batch);
  if (which == 0) {
    const size_t bytes = (size_t)W::WARPS * W::STRIDE * sizeof(double2);
    static AttrOnce attr;
    if (!attr.ensure(rows_tt_w<W>, bytes)) return -1;
    launch_k(rows_tt_w<W>, grid, 32 * W::WARPS, bytes, s, a);
  } else {
    const size_t bytes = (size_t)W::WARPS * W::RLS * sizeof(double2);
    static AttrOnce attr;
    if (!attr.ensure(rows_t_axpy_w<W>, bytes)) return -1;
    launch_k(rows_t_axpy_w<W>, grid, 32 * W::WARPS, bytes, s, a);
  }
  return (int)grid.x;
}

// Warp-owned row kernels of the separable pipeline for 1024- and 256-point
// rows (q2 <= 15); -1 when the shape is not theirs.
int launch_rows_w(int which, const SpecArgs& a, cudaStream_t s) {
  if (a.q2 > 15 || !conv_sep_supported(a.q2)) return -1;
  if (a.n2 == 1024 && a.blue2.N == W1023::N) return launch_rows_w_t<W1023>(which, a, s);
  if (a.n2 == 256 && a.blue2.N == W255::N && kW255) return launch_rows_w_t<W255>(which, a, s);
  return -1;
}

}  // namespace dbx
