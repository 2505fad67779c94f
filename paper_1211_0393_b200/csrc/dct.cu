// dct.cu — CosineIII algebra transforms for reflective boundary conditions
// (the paper's comparison path): the orthonormal
// R_m(s,t) = sqrt((2 - delta_{s,0})/m) cos(s (2t+1) pi / 2m) of
// cosine3_forward (FFTW REDFT10) and R_m^T of cosine3_inverse (REDFT01),
// transforms.hpp:88-110, along the rows of a batch, two rows per complex
// m-point FFT (Makhoul's reordering):
//
//   forward: v_n = x_{2n}, v_{m-1-n} = x_{2n+1};  V = FFT(v);
//            X_k = c_k Re(w_k V_k),  w_k = e^{-i pi k / 2m}
//   inverse: Y_k = X_k / c_k;  V_k = conj(w_k) (Y_k - i Y_{m-k})  (Y_m = 0);
//            v = IFFT(V) / m;  x_{2n} = v_n, x_{2n+1} = v_{m-1-n}
//
// Rows a, b share one FFT of v^a + i v^b (split by conjugate symmetry for the
// forward, packed as V^a + i V^b for the inverse).  The outputs overwrite the
// FFT line in place; the epilogue is the shared one (store / Hadamard by the
// filter grid / x update with norms).  Columns run on transposed images.
#include <cuda_runtime.h>

#include "spectral_common.cuh"

namespace dbx {

namespace {

template <int M>
struct DctCfg {
  static constexpr int T = line_threads(M, 8);
  static constexpr int G = lines_for(M, kDstBudget, 8);  // FFT lines (row pairs) per CTA
  static constexpr int NT = T * G;
  static constexpr int LINE = padded_len(M);
  static constexpr int TWN = fft::twiddles_needed(M);
  static constexpr size_t base = (size_t)G * LINE * 16;
  static constexpr bool TW = base + (size_t)TWN * 16 <= kSmemCap;
  static constexpr size_t bytes = base + (TW ? (size_t)TWN * 16 : 0);
  static constexpr int PK = (M / 2 + 1 + T - 1) / T;  // forward split items per thread
  static constexpr int PN = (M + T - 1) / T;          // inverse unpack items per thread
};

__device__ __forceinline__ int dct_perm(int n, int m) {  // position n of v holds x_{perm(n)}
  return n < (m + 1) / 2 ? 2 * n : 2 * (m - 1 - n) + 1;
}

template <int M>
__global__ void __launch_bounds__(DctCfg<M>::NT) dct_rows(SpecArgs a) {
  DBX_PDL_WAIT();
  using C = DctCfg<M>;
  constexpr int T = C::T, G = C::G, NT = C::NT;
  const int b = blockIdx.y;
  if (a.st && a.st[b].done) return;
  extern __shared__ double2 sm[];
  __shared__ double red[32];
  const int g = threadIdx.x / T, t = threadIdx.x - g * T;
  double2* buf = sm + g * C::LINE;
  const BlueTables& bt = a.blue2;
  const double2* tw = stage_twiddles<M, C::TW>(sm + G * C::LINE, bt.tw);
  const int n1 = a.n1;
  const size_t N = (size_t)n1 * M;
  const int ra = blockIdx.x * 2 * G + 2 * g;
  const bool la = ra < n1, lb = ra + 1 < n1;
  const double* in = resolve_ptr(a.in, a.st, a.insel, b, a.batch, N);
  const double* xa = in + (size_t)(la ? ra : 0) * M;
  const double* xb = in + (size_t)(lb ? ra + 1 : 0) * M;
  const bool fwd = a.kind1 > 0;
  const int bar = G > 1 ? 1 + g : 0;
  const double c0 = bt.c0, c = bt.scale;
  double* oa = reinterpret_cast<double*>(buf);
  double* ob = oa + M;
  if (fwd) {
    for (int n = t; n < M; n += T) {
      const int j = dct_perm(n, M);
      buf[pad<M>(n)] = make_double2(la ? xa[j] : 0.0, lb ? xb[j] : 0.0);
    }
    cp_async_wait_all();
    __syncthreads();
    fft::fft<M, -1, T>(buf, tw, t, bar);
    // split the two rows' spectra; k and m-k from one pair of loads
    double r[C::PK][4];
#pragma unroll
    for (int i = 0; i < C::PK; ++i) {
      const int k = t + i * T;
      if (k <= M / 2) {
        const int m = k == 0 ? 0 : M - k;
        const double2 zk = buf[pad<M>(k)], zm = buf[pad<M>(m)];
        const double2 A = make_double2(0.5 * (zk.x + zm.x), 0.5 * (zk.y - zm.y));
        const double2 B = make_double2(0.5 * (zk.y + zm.y), 0.5 * (zm.x - zk.x));
        const double2 wk = __ldg(bt.chirp + k), wm = __ldg(bt.chirp + m);
        const double ck = k == 0 ? c0 : c;
        r[i][0] = ck * (wk.x * A.x - wk.y * A.y);  // X^a_k
        r[i][1] = ck * (wk.x * B.x - wk.y * B.y);  // X^b_k
        r[i][2] = c * (wm.x * A.x + wm.y * A.y);   // X^a_{m-k} = c Re(w_{m-k} conj(A_k))
        r[i][3] = c * (wm.x * B.x + wm.y * B.y);
      }
    }
    fft::line_sync(bar, T);
#pragma unroll
    for (int i = 0; i < C::PK; ++i) {
      const int k = t + i * T;
      if (k <= M / 2) {
        oa[k] = r[i][0];
        ob[k] = r[i][1];
        if (k != 0 && k != M - k) {
          oa[M - k] = r[i][2];
          ob[M - k] = r[i][3];
        }
      }
    }
  } else {
    const double ic0 = 1.0 / c0, ic = 1.0 / c;
    for (int k = t; k < M; k += T) {
      const double2 w = __ldg(bt.chirp + k);
      const double sk = k == 0 ? ic0 : ic;
      const double pa = la ? xa[k] * sk : 0.0, pb = lb ? xb[k] * sk : 0.0;
      const double qa = (k == 0 || !la) ? 0.0 : -xa[M - k] * ic, qb = (k == 0 || !lb) ? 0.0 : -xb[M - k] * ic;
      // conj(w) (p + i q)
      const double2 Wa = make_double2(pa * w.x + qa * w.y, qa * w.x - pa * w.y);
      const double2 Wb = make_double2(pb * w.x + qb * w.y, qb * w.x - pb * w.y);
      buf[pad<M>(k)] = make_double2(Wa.x - Wb.y, Wa.y + Wb.x);
    }
    cp_async_wait_all();
    __syncthreads();
    fft::fft<M, +1, T>(buf, tw, t, bar);
    const double im = 1.0 / (double)M;
    double2 v[C::PN];
#pragma unroll
    for (int i = 0; i < C::PN; ++i) {
      const int n = t + i * T;
      if (n < M) v[i] = buf[pad<M>(n)];
    }
    fft::line_sync(bar, T);
#pragma unroll
    for (int i = 0; i < C::PN; ++i) {
      const int n = t + i * T;
      if (n < M) {
        const int j = dct_perm(n, M);
        oa[j] = v[i].x * im;
        ob[j] = v[i].y * im;
      }
    }
  }
  __syncthreads();
  Epi e = make_epi(a, b, N);
  for (int hh = 0; hh < 2; ++hh) {
    const int rr = ra + hh;
    if (rr >= n1) continue;
    const double* o = hh ? ob : oa;
    for (int k = t; k < M; k += T) e.put((size_t)rr * M + k, o[k]);
  }
  write_partials<NT>(a, e, red, b);
}

template <int L>
int dct_launch(const SpecArgs& a, cudaStream_t s) {
  using C = DctCfg<L>;
  static AttrOnce attr;
  if (!attr.ensure(dct_rows<L>, C::bytes)) return -1;
  dim3 grid((a.n1 + 2 * C::G - 1) / (2 * C::G), a.batch);
  launch_k(dct_rows<L>, grid, C::NT, C::bytes, s, a);
  return (int)grid.x;
}

}  // namespace

#define DBX_DCT_LIST(X)                                                                              \
  X(4) X(6) X(8) X(10) X(12) X(16) X(24) X(32) X(48) X(64) X(96) X(128) X(256) X(512) X(1024) X(2048) \
  X(4096) X(8192)

int dct_supported_len(int m) {
#define X(L) if (m == (L)) return (L);
  DBX_DCT_LIST(X)
#undef X
  return 0;
}

int launch_dct_rows(const SpecArgs& a, cudaStream_t s) {
  const int m = a.n2;
#define X(L) if (m == (L)) return dct_launch<L>(a, s);
  DBX_DCT_LIST(X)
#undef X
  return -1;
}

}  // namespace dbx
