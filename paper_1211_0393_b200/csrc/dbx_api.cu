// dbx_api.cu — host side of the C-ABI (include/dbx.h): plan lifetime, argument
// validation with the reference's error semantics, host/device staging, the
// dense AR transform matrices, and the Landweber driver (captured as one CUDA
// graph per run shape).  No CPU compute path exists: every numerical result is
// produced by the sm_100a kernels in blur.cu / gemm.cu / solver_kernels.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <future>
#include <memory>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dbx.h"
#include "dbx_internal.h"
#include "spectral.h"
#include "tables.h"

using namespace dbx;

// Off by default: measured A/B (profiles/r02_pdl_ab.txt) put every config
// behind plain stream order with it on (C1 1468 vs 1564, C2 2972 vs 3695, C3
// 22562 vs 23196 Mpx-it/s): the dependents' early-resident CTAs cost more than
// the launch gaps they hide.  DBX_PDL=1 turns it on.
bool dbx::pdl_enabled() {
  static const bool on = [] { const char* e = getenv("DBX_PDL"); return e && e[0] == '1'; }();
  return on;
}

namespace {

thread_local std::string g_err;

struct InvalidArg : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct Diverged : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// core.hpp:26-28 detail::require
inline void require(bool c, const std::string& what) {
  if (!c) throw InvalidArg(what);
}

inline void ck(cudaError_t e, const char* where) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw CudaErr(std::string(where) + ": " + cudaGetErrorString(e));
  }
}

template <typename F>
int guarded(F&& f) {
  try {
    f();
    g_err.clear();
    return DBX_OK;
  } catch (const InvalidArg& e) {
    g_err = e.what();
    return DBX_EINVAL;
  } catch (const Diverged& e) {
    g_err = e.what();
    return DBX_EDIVERGED;
  } catch (const CudaErr& e) {
    g_err = e.what();
    return DBX_ECUDA;
  } catch (const std::exception& e) {
    g_err = e.what();
    return DBX_ECUDA;
  }
}

// Device (or managed) memory usable in place by kernels on the CURRENT device
// (every entry point calls set_dev() first).  Device memory of another GPU
// is refused instead of being read through peer mappings or faulting.
bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes at;
  if (cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (at.type == cudaMemoryTypeDevice) {
    int cur = 0;
    cudaGetDevice(&cur);
    if (at.device != cur)
      throw InvalidArg("device pointer on GPU " + std::to_string(at.device) + ", plan on GPU " +
                       std::to_string(cur));
    return true;
  }
  return at.type == cudaMemoryTypeManaged;
}

struct DevBuf {
  double* p = nullptr;
  size_t n = 0;
  void ensure(size_t count) {
    if (count <= n) return;
    if (p) cudaFree(p);
    p = nullptr;
    ck(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(double)), "cudaMalloc");
    n = count;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
};

// Dense T~_n, T_n, Q_n with integer-reduced sine arguments:
// Q_m(s,t) = sqrt(2/(m+1)) sin(pi ((s t) mod 2(m+1)) / (m+1)), long double.
std::vector<long double> sine_table(long m) {
  const long N2 = 2 * (m + 1);
  std::vector<long double> tab((size_t)N2);
  const long double pi = 3.141592653589793238462643383279502884L;
  for (long e = 0; e < N2; ++e) tab[(size_t)e] = sinl(pi * (long double)e / (long double)(m + 1));
  return tab;
}

// Q_m as an m x m matrix (1-based s,t), long double entries.
void fill_q(long m, std::vector<long double>& q) {
  const auto tab = sine_table(m);
  const long N2 = 2 * (m + 1);
  const long double sc = sqrtl(2.0L / (long double)(m + 1));
  q.assign((size_t)(m * m), 0.0L);
  for (long s = 1; s <= m; ++s)
    for (long t = 1; t <= m; ++t) q[(size_t)((s - 1) * m + (t - 1))] = sc * tab[(size_t)((s * t) % N2)];
}

// transforms.hpp:135-144 (p and alpha exactly as the reference computes them)
void ar_params(long n, std::vector<double>& p, double& alpha) {
  p.assign((size_t)(n - 2), 0.0);
  double sq = 0.0;
  for (long j = 1; j <= n - 2; ++j) p[(size_t)(j - 1)] = 1.0 - (double)j / (double)(n - 1);
  for (double v : p) sq += v * v;
  alpha = std::sqrt(1.0 + sq);
}

// dense matrix slots: the DBX_KIND_* values, plus slot 0 for R^T (inverse cosine)
constexpr int MK_COSINV = 0;

// kind: DBX_KIND_SINEI -> Q_n ; DBX_KIND_AR -> T_n ; DBX_KIND_ARINV -> T~_n ;
// DBX_KIND_COSINE3 -> R_n ; MK_COSINV -> R_n^T (transforms.hpp:88-110)
std::vector<double> dense_transform(int kind, long n) {
  std::vector<double> M((size_t)(n * n), 0.0);
  if (kind == DBX_KIND_COSINE3 || kind == MK_COSINV) {
    const long double pi = 3.141592653589793238462643383279502884L;
    for (long s = 0; s < n; ++s)
      for (long t = 0; t < n; ++t) {
        const long e = (s * (2 * t + 1)) % (4 * n);  // exact reduction of s (2t+1) pi / 2n
        const long double v = sqrtl((s == 0 ? 1.0L : 2.0L) / (long double)n) * cosl(pi * (long double)e / (long double)(2 * n));
        M[(size_t)(kind == MK_COSINV ? t * n + s : s * n + t)] = (double)v;
      }
    return M;
  }
  if (kind == DBX_KIND_SINEI) {
    std::vector<long double> q;
    fill_q(n, q);
    for (size_t i = 0; i < q.size(); ++i) M[i] = (double)q[i];
    return M;
  }
  const long m = n - 2;
  std::vector<long double> q;
  fill_q(m, q);
  std::vector<double> p;
  double alpha;
  ar_params(n, p, alpha);
  for (long s = 0; s < m; ++s)
    for (long t = 0; t < m; ++t) M[(size_t)((s + 1) * n + (t + 1))] = (double)q[(size_t)(s * m + t)];
  if (kind == DBX_KIND_AR) {
    // dense_ar_forward block form: first/last columns = normalised ramps
    const double inv_a = 1.0 / alpha;
    M[0] = inv_a;
    M[(size_t)(n * n - 1)] = inv_a;
    for (long j = 0; j < m; ++j) {
      M[(size_t)((1 + j) * n)] = inv_a * p[(size_t)j];
      M[(size_t)((1 + j) * n + (n - 1))] = inv_a * p[(size_t)(m - 1 - j)];
    }
  } else {
    // dense_ar_inverse block form: [alpha 0 0; -Qp Q -QJp; 0 0 alpha]
    M[0] = alpha;
    M[(size_t)(n * n - 1)] = alpha;
    for (long s = 0; s < m; ++s) {
      long double qp = 0.0L, qjp = 0.0L;
      for (long t = 0; t < m; ++t) {
        qp += q[(size_t)(s * m + t)] * (long double)p[(size_t)t];
        qjp += q[(size_t)(s * m + t)] * (long double)p[(size_t)(m - 1 - t)];
      }
      M[(size_t)((1 + s) * n)] = -(double)qp;
      M[(size_t)((1 + s) * n + (n - 1))] = -(double)qjp;
    }
  }
  return M;
}

std::vector<double> transpose(const std::vector<double>& a, long n) {
  std::vector<double> t(a.size());
  for (long i = 0; i < n; ++i)
    for (long j = 0; j < n; ++j) t[(size_t)(j * n + i)] = a[(size_t)(i * n + j)];
  return t;
}

// Launcher result check: a negative CTA count means the size is not compiled
// or its shared-memory plan does not fit this device.
thread_local const char* t_last_kernel = nullptr;  // name of the last lc() launch (per-kernel timing)
inline int lc(int rc, const char* what) {
  if (rc < 0) throw CudaErr(std::string(what) + ": launch configuration unsupported on this device");
  t_last_kernel = what;
  return rc;
}

enum KClass { KC_BLUR_ADJ = 0, KC_BLUR = 1, KC_TRANSFORM = 2, KC_FINALIZE = 3, KC_NUM = 4 };

}  // namespace

constexpr double kSepTol = 1e-14;  // rank-1 test: max |w - a b^T| / max |w|

struct dbx_plan {
  int n1 = 0, n2 = 0, batch = 0, q1 = 0, q2 = 0, device = 0;
  size_t N = 0;
  std::vector<double> taps;
  cudaStream_t stream = nullptr;
  double* w_A = nullptr;   // weights of A (rotate180 of taps)
  double* w_At = nullptr;  // weights of A' (taps)
  double* sym = nullptr;   // symmetrised taps (psf.hpp:71-85)
  double* d = nullptr;     // filter grid (one shared, or one per image for an alpha sweep)
  size_t d_cap = 0;        // doubles allocated at d
  size_t dstride = 0;      // 0: shared grid; N: per-image grids (dbx_precond_build_sweep)
  uint64_t dgen = 0;       // filter generation (part of the graph-cache key)
  bool have_d = false;
  int conv = DBX_CONV_AUTO;
  // dense transform matrices [kind][0 col-matrix (n1), 1 row-matrix^T (n2)]
  double* mats[5][2] = {};
  DevBuf g, f, r, s, u, X3, in, out, part, rre, res, xh;
  ImgState* st = nullptr;
  int part_cap = 0;
  int64_t launches = 0;
  bool timing = false;
  double kms[KC_NUM] = {};
  int kcount[KC_NUM] = {};
  std::vector<cudaEvent_t> evpool;
  size_t evused = 0;
  std::vector<std::pair<int, size_t>> evrecs;
  std::vector<const char*> evnames;                       // kernel name per record (lc() name, else the class)
  std::vector<std::pair<std::string, std::pair<double, int>>> kprof;  // per kernel name: ms, launches
  // graph cache
  cudaGraphExec_t gexec = nullptr;
  std::string gkey;
  int64_t glaunches = 0;
  bool fusion = true;  // fused row pipelines when compiled for the sizes
  int bc = DBX_BC_ANTIREFLECTIVE;  // BoundaryCondition of the blur (and the preconditioner algebra)
  int last_fused = 0;  // pipeline of the last landweber run: 0 separate passes, 1 fused, 2 fused separable
  // ---- FFT-form state ----
  int dst = DBX_DST_AUTO;
  bool conv_ready = false;
  int L1 = 0, L2 = 0, Lh = 0;
  double *tw1 = nullptr, *tw2 = nullptr, *HA = nullptr, *HAt = nullptr;
  // rank-1 mask: separable column pass (conv_col_sep) tables for A (rotated
  // mask) and A' (mask); sep_ok when both factor within kSepTol
  double *sepA_a = nullptr, *sepA_b = nullptr, *sepAt_a = nullptr, *sepAt_b = nullptr;
  double *sepA_r = nullptr, *sepAt_r = nullptr;  // row factors (direct row passes, separable fused pipeline)
  std::vector<double> sepA_a_h, sepAt_a_h;         // host copies of the column taps (kernel-parameter taps)
  std::vector<double> sepA_r_h, sepAt_r_h;         // host copies of the row taps (ConvTables::sepr_v)
  bool sep_ok = false;
  double sep_resid = 1.0;
  DevBuf zb, yb, dT;  // dT: filter grid transposed (fused column pass)
  DevBuf fincnt;      // per-image arrival counters of the last-block finalize (fused pipelines)
  DevBuf cg_p, cg_q, cg_s, cg_z, cg_zero, cg_part, cg_sc;  // CGLS state (dbx_cgls_run)
  struct Blue {
    bool ready = false;
    double *tw = nullptr, *chirp = nullptr, *bhat = nullptr, *p = nullptr, *sn = nullptr;
    BlueTables t;
  } blue[2][2];  // [axis 0 = columns (n1), 1 = rows (n2)][0 = AR kinds, 1 = SineI]
  std::vector<double*> owned;

  ~dbx_plan() {
    if (gexec) cudaGraphExecDestroy(gexec);
    for (auto e : evpool) cudaEventDestroy(e);
    for (auto& km : mats)
      for (auto p : km)
        if (p) cudaFree(p);
    for (double* p : {w_A, w_At, sym, d})
      if (p) cudaFree(p);
    for (double* p : owned) cudaFree(p);
    if (st) cudaFree(st);
    for (DevBuf* b : {&g, &f, &r, &s, &u, &X3, &in, &out, &part, &rre, &res, &xh, &zb, &yb, &dT, &fincnt, &cg_p, &cg_q,
                      &cg_s, &cg_z, &cg_zero, &cg_part, &cg_sc})
      b->release();
    if (stream) cudaStreamDestroy(stream);
  }

  double* upload_owned(const std::vector<double>& h) {
    double* p = upload(h);
    owned.push_back(p);
    return p;
  }
  const int* upload_owned_int(const std::vector<int>& h) {
    int* p = nullptr;
    ck(cudaMalloc(&p, h.size() * sizeof(int)), "cudaMalloc");
    ck(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(int), cudaMemcpyHostToDevice, stream), "upload");
    ck(cudaStreamSynchronize(stream), "upload sync");
    owned.push_back(reinterpret_cast<double*>(p));
    return p;
  }

  // ---- engine selection ----
  // Conv: the reference switches to FFT correlation for q > 7 (blur.hpp:70,
  // 79-82); AUTO follows that cutover whenever a compiled FFT length fits.
  int conv_len(int n, int q) const { return conv_supported_len(n + 2 * q + (n + 2 * q) % 2); }
  // Below the cutover AUTO still takes the FFT engine when it unlocks the
  // fused preconditioned pipeline for this shape (fused.cu): C1 (256^2, q = 7)
  // runs 6 fused launches per iteration instead of the direct stencil's
  // separate passes, 1.9x faster end to end, at the same <= 1e-10 parity.
  bool use_fft_conv() const {
    if (conv == DBX_CONV_DIRECT) return false;
    const bool fits = conv_len(n1, q1) > 0 && conv_len(n2, q2) > 0;
    if (conv == DBX_CONV_FFT || conv == DBX_CONV_FFT_DENSE) return fits;
    return fits && (q1 > 7 || q2 > 7 || fused_shape());
  }
  bool fused_shape() const {
    if (bc != DBX_BC_ANTIREFLECTIVE || n1 != n2 || n1 < 3 || conv_len(n2, q2) <= 0) return false;
    int M = 0;
    const int core = dst_core(n1 - 1, &M);
    return (core == CORE_DIRECT || core == CORE_BLUE || core == CORE_PFA) &&
           fused_supported(conv_len(n2, q2), M, core == CORE_BLUE);
  }
  // DST core and DFT length M for an N-point DFT: direct (N compiled: prime
  // factors <= 31), Bluestein (compiled power of two M >= 2N-1), Rader (N
  // prime, N-1 compiled; e.g. 8191 for C5).  DBX_DST_RADER forces Rader.
  int dst_core(int N, int* M) const {
    // DBX_DST_PFA=0: Bluestein instead of the prime-factor core (A/B, tests)
    static const bool pfa_off = [] { const char* e = getenv("DBX_DST_PFA"); return e && e[0] == '0'; }();
    if (dst != DBX_DST_RADER) {
      if (direct_supported_len(N)) { *M = N; return CORE_DIRECT; }
      if (!pfa_off && pfa_supported_len(N)) { *M = N; return CORE_PFA; }
      const int Mb = blue_supported_len(2 * N - 1 < 16 ? 16 : 2 * N - 1);
      if (Mb) { *M = Mb; return CORE_BLUE; }
    }
    if (N > 2 && is_prime(N) && rader_supported_len(N - 1)) { *M = N - 1; return CORE_RADER; }
    return -1;
  }
  // CosineIII transforms (reflective BCs): FFT form when both line lengths are
  // compiled DCT lengths (dct.cu), else the dense GEMM form.
  bool use_fft_dct() const {
    return dst != DBX_DST_DENSE && dct_supported_len(n1) && dct_supported_len(n2);
  }
  struct Dct {
    bool ready = false;
    BlueTables t;
  } dct[2];
  const BlueTables& dct_tables(int axis) {
    Dct& D = dct[axis];
    if (!D.ready) {
      const int m = axis == 0 ? n1 : n2;
      std::vector<double> w(2 * (size_t)m);
      const long double pi = 3.141592653589793238462643383279502884L;
      for (long k = 0; k < m; ++k) {  // w_k = exp(-i pi k / 2m)
        w[2 * k] = (double)cosl(pi * (long double)k / (long double)(2 * m));
        w[2 * k + 1] = -(double)sinl(pi * (long double)k / (long double)(2 * m));
      }
      D.t.tw = reinterpret_cast<const double2*>(upload_owned(twiddles(m)));
      D.t.chirp = reinterpret_cast<const double2*>(upload_owned(w));
      D.t.scale = (double)sqrtl(2.0L / (long double)m);
      D.t.c0 = (double)sqrtl(1.0L / (long double)m);
      D.t.n = m; D.t.N = m; D.t.M = m;
      D.ready = true;
    }
    return D.t;
  }

  // DBX_DST_TDT=0: the column half of D as two row passes (A/B switch)
  static bool dst_tdt_fused() {
    static const bool on = [] { const char* e = getenv("DBX_DST_TDT"); return !(e && e[0] == '0'); }();
    return on;
  }
  // Transposed stores from dst_rows instead of explicit transposes between the
  // row passes of D (C4 7724 -> 8037, C5 9385 -> 9650 Mpx-it/s,
  // profiles/r03_dst_tout_ab.txt); DBX_DST_TOUT=0 restores the transposes (A/B)
  static bool dst_tout() {
    static const bool on = [] { const char* e = getenv("DBX_DST_TOUT"); return !(e && e[0] == '0'); }();
    return on;
  }
  bool use_fft_dst(bool sine) const {
    if (dst == DBX_DST_DENSE) return false;
    const int N1 = sine ? n1 + 1 : n1 - 1, N2 = sine ? n2 + 1 : n2 - 1;
    int M = 0;
    return N1 >= 2 && N2 >= 2 && dst_core(N1, &M) >= 0 && dst_core(N2, &M) >= 0;
  }

  // direct separable blur in the separate passes (rank-1 mask, compiled tap
  // counts; plain Landweber's AXPY epilogue keeps the FFT form).
  // DBX_SEP_DIRECT=0 disables it (A/B and tests).
  bool sep_direct(int mode) const {
    static const bool off = [] { const char* e = getenv("DBX_SEP_DIRECT"); return e && e[0] == '0'; }();
    return !off && sep_ok && conv != DBX_CONV_FFT_DENSE && mode != BLUR_AXPY && conv_sep_supported(q1) &&
           rows_sep_supported(q2);
  }

  // kernel spectrum of A (adjoint = false) or A' for the column pass, and the
  // separable tables when the mask is rank 1 (unless DBX_CONV_FFT_DENSE)
  void set_kernel(ConvTables& c, bool adjoint) const {
    c.H = reinterpret_cast<const double2*>(adjoint ? HAt : HA);
    const bool sep = sep_ok && conv != DBX_CONV_FFT_DENSE;
    c.sepa = sep ? (adjoint ? sepAt_a : sepA_a) : nullptr;
    c.sepb = sep ? reinterpret_cast<const double2*>(adjoint ? sepAt_b : sepA_b) : nullptr;
    c.sepr = sep ? (adjoint ? sepAt_r : sepA_r) : nullptr;
    c.sepa_host = sep ? (adjoint ? sepAt_a_h.data() : sepA_a_h.data()) : nullptr;
    if (sep) {
      const std::vector<double>& r = adjoint ? sepAt_r_h : sepA_r_h;
      for (size_t t = 0; t < r.size() && t < 31; ++t) c.sepr_v[t] = r[t];
    }
  }

  void ensure_conv() {
    if (conv_ready) return;
    L1 = conv_len(n1, q1);
    L2 = conv_len(n2, q2);
    Lh = L2 / 2 + 1;
    tw1 = upload_owned(twiddles(L1));
    tw2 = upload_owned(twiddles(L2));
    const size_t nt = taps.size();
    std::vector<double> rot(taps.rbegin(), taps.rend());
    // k2-major spectra; for the CT column core (kConvCt) each column k2 in
    // the digit-reversed order of the in-place DIF output
    auto ct_order = [&](std::vector<double> h) {
      if (!kConvCt) return h;
      std::vector<double> o(h.size());
      const int Lh_ = L2 / 2 + 1;
      for (int k2 = 0; k2 < Lh_; ++k2)
        for (int p = 0; p < L1; ++p) {
          const size_t src = 2 * ((size_t)k2 * L1 + fft::ct_freq_of_pos(L1, p)), dst = 2 * ((size_t)k2 * L1 + p);
          o[dst] = h[src];
          o[dst + 1] = h[src + 1];
        }
      return o;
    };
    HA = upload_owned(ct_order(conv_spectrum(rot.data(), q1, q2, L1, L2)));
    HAt = upload_owned(ct_order(conv_spectrum(taps.data(), q1, q2, L1, L2)));
    // separable column pass for a rank-1 mask (factorisation residual within
    // kSepTol of the largest tap: rounding level, far below the 1e-10 parity)
    if (q1 > 0 && conv_sep_supported(q1)) {
      std::vector<double> aA, bA, aAt, bAt, rwA, rwAt;
      double rA = 1.0, rAt = 1.0;
      if (rank1_factor(rot.data(), q1, q2, L2, kSepTol, aA, bA, &rA, &rwA) &&
          rank1_factor(taps.data(), q1, q2, L2, kSepTol, aAt, bAt, &rAt, &rwAt)) {
        sepA_a = upload_owned(aA);
        sepA_b = upload_owned(bA);
        sepAt_a = upload_owned(aAt);
        sepAt_b = upload_owned(bAt);
        sepA_r = upload_owned(rwA);
        sepAt_r = upload_owned(rwAt);
        sepA_a_h = aA;
        sepAt_a_h = aAt;
        sepA_r_h = rwA;
        sepAt_r_h = rwAt;
        sep_ok = true;
      }
      sep_resid = std::max(rA, rAt);
    }
    (void)nt;
    zb.ensure((size_t)batch * n1 * Lh * 2);
    yb.ensure((size_t)batch * n1 * y_stride(Lh) * 2);
    conv_ready = true;
  }

  const BlueTables& blue_tables(int axis, bool sine) {
    Blue& B = blue[axis][sine ? 1 : 0];
    if (!B.ready) {
      const int n = axis == 0 ? n1 : n2;
      const int N = sine ? n + 1 : n - 1;
      int M = 0;
      const int core = dst_core(N, &M);
      require(core >= 0, "no FFT-form DST for this line length");
      int pn1 = 0, pn2 = 0;
      if (core == CORE_PFA) pfa_factors(N, &pn1, &pn2);
      const BlueHost h = core == CORE_RADER ? rader(n, sine)
                         : core == CORE_PFA ? pfa(n, sine, pn1, pn2) : bluestein(n, sine, M);
      B.tw = upload_owned(h.tw);
      B.chirp = upload_owned(h.chirp);
      B.bhat = upload_owned(h.bhat);
      B.p = upload_owned(h.p);
      B.sn = upload_owned(h.sn);
      B.t.sn = B.sn;
      if (core == CORE_RADER || core == CORE_PFA) {
        B.t.dlog = upload_owned_int(h.dlog);
        B.t.ridx = upload_owned_int(h.ridx);
      }
      B.t.core = core;
      B.t.tw = reinterpret_cast<const double2*>(B.tw);
      B.t.chirp = reinterpret_cast<const double2*>(B.chirp);
      B.t.bhat = reinterpret_cast<const double2*>(B.bhat);
      if (!h.bct.empty()) B.t.bct = reinterpret_cast<const double2*>(upload_owned(h.bct));
      if (!h.bctT.empty()) B.t.bctT = reinterpret_cast<const double2*>(upload_owned(h.bctT));
      if (!h.tw1t.empty()) B.t.tw1t = reinterpret_cast<const double2*>(upload_owned(h.tw1t));
      B.t.p = B.p;
      B.t.alpha = h.alpha;
      B.t.rinv = n > 1 ? 1.0 / (double)(n - 1) : 1.0;
      B.t.scale = h.scale;
      B.t.n = h.n;
      B.t.N = h.N;
      B.t.M = h.M;
      B.ready = true;
    }
    return B.t;
  }

  // prepare everything a run needs before graph capture (no allocation inside)
  void prepare(bool precond) {
    if (use_fft_conv()) ensure_conv();
    if (precond && bc == DBX_BC_REFLECTIVE) {
      if (use_fft_dct()) {
        dct_tables(0);
        dct_tables(1);
      } else {
        matrix(DBX_KIND_COSINE3, 0); matrix(DBX_KIND_COSINE3, 1);
        matrix(MK_COSINV, 0); matrix(MK_COSINV, 1);
      }
    } else if (precond) {
      if (use_fft_dst(false)) {
        blue_tables(0, false);
        blue_tables(1, false);
      } else {
        matrix(DBX_KIND_ARINV, 0); matrix(DBX_KIND_ARINV, 1);
        matrix(DBX_KIND_AR, 0); matrix(DBX_KIND_AR, 1);
      }
    }
  }

  SpecArgs spec_base(const ImgState* stp, Partials pt) const {
    SpecArgs a;
    a.n1 = n1; a.n2 = n2; a.q1 = q1; a.q2 = q2; a.batch = batch;
    a.st = stp; a.part = pt;
    a.dstride = dstride;
    a.bc = bc;
    return a;
  }

  void set_dev() const { ck(cudaSetDevice(device), "cudaSetDevice"); }

  void ensure_d(size_t count) {
    ++dgen;  // every filter (re)build: captured graphs bake d, dT and dstride in
    if (d && d_cap >= count) return;
    if (d) cudaFree(d);
    d = nullptr;
    ck(cudaMalloc(&d, count * sizeof(double)), "cudaMalloc");
    d_cap = count;
  }

  // Ordered on the plan's (non-blocking) stream: a plain cudaMemcpy from
  // pageable memory may return before its DMA lands, which would race the
  // next kernel on this stream.
  double* upload(const std::vector<double>& h) {
    double* p = nullptr;
    ck(cudaMalloc(&p, h.size() * sizeof(double)), "cudaMalloc");
    ck(cudaMemcpyAsync(p, h.data(), h.size() * sizeof(double), cudaMemcpyHostToDevice, stream), "upload");
    ck(cudaStreamSynchronize(stream), "upload sync");
    return p;
  }

  double* matrix(int kind, int which) {
    if (!mats[kind][which]) {
      const long n = which == 0 ? n1 : n2;
      auto M = dense_transform(kind, n);
      if (which == 1) M = transpose(M, n);
      mats[kind][which] = upload(M);
    }
    return mats[kind][which];
  }

  // ---- launch bookkeeping (optional per-class CUDA-event timing) ----
  void ev_begin(int cls) {
    ++launches;
    if (!timing) return;
    if (evused + 2 > evpool.size()) {
      for (int i = 0; i < 64; ++i) {
        cudaEvent_t e;
        ck(cudaEventCreate(&e), "cudaEventCreate");
        evpool.push_back(e);
      }
    }
    ck(cudaEventRecord(evpool[evused], stream), "cudaEventRecord");
    evrecs.push_back({cls, evused});
    evused += 2;
    t_last_kernel = nullptr;
  }
  void ev_end() {
    if (!timing) return;
    ck(cudaEventRecord(evpool[evrecs.back().second + 1], stream), "cudaEventRecord");
    static const char* cls_name[KC_NUM] = {"blur_adjoint", "blur", "ar_transform", "finalize"};
    evnames.push_back(t_last_kernel ? t_last_kernel : cls_name[evrecs.back().first]);
  }
  void ev_collect() {
    if (!timing) return;
    ck(cudaStreamSynchronize(stream), "sync");
    for (int i = 0; i < KC_NUM; ++i) kms[i] = 0.0, kcount[i] = 0;
    kprof.clear();
    for (size_t i = 0; i < evrecs.size(); ++i) {
      const auto& rc = evrecs[i];
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, evpool[rc.second], evpool[rc.second + 1]), "elapsed");
      kms[rc.first] += ms;
      kcount[rc.first] += 1;
      const std::string nm = std::string(i < evnames.size() ? evnames[i] : "?") + "#" + std::to_string(rc.first);
      auto it = std::find_if(kprof.begin(), kprof.end(), [&](const auto& e) { return e.first == nm; });
      if (it == kprof.end()) kprof.push_back({nm, {(double)ms, 1}});
      else it->second.first += ms, it->second.second += 1;
    }
    evrecs.clear();
    evnames.clear();
    evused = 0;
  }

  void check_launch() { ck(cudaGetLastError(), "kernel launch"); }

  int blur(const double* x, int xsel, double* y, int ysel, bool adjoint, int mode,
           const double* gg, const double* xold, int xoldsel, const double* ff, double tau,
           const ImgState* stp, Partials pt, int cls) {
    if (use_fft_conv()) {
      ensure_conv();
      if (sep_direct(mode)) {
        // rank-1 mask: direct row pass + direct column pass (2 (2q+1) flops
        // per pixel, no FFTs), residual / store fused into the column pass
        SpecArgs a = spec_base(stp, pt);
        set_kernel(a.conv, adjoint);
        a.zbuf = reinterpret_cast<double2*>(zb.p);
        a.in = x; a.insel = xsel;
        a.out = y; a.outsel = ysel;
        a.g = gg;
        ev_begin(cls);
        lc(launch_rows_sep_seg(a, stream), "rows_sep_seg");
        const int ctas = lc(launch_cols_sep_epi(a, mode == BLUR_RESID ? 1 : 0, stream), "cols_sep_real");
        ev_end();
        launches += 2;
        check_launch();
        return ctas;
      }
      SpecArgs a = spec_base(stp, pt);
      a.conv.tw1 = reinterpret_cast<const double2*>(tw1);
      a.conv.tw2 = reinterpret_cast<const double2*>(tw2);
      set_kernel(a.conv, adjoint);
      a.conv.L1 = L1; a.conv.L2 = L2; a.conv.Lh = Lh;
      a.zbuf = reinterpret_cast<double2*>(zb.p);
      a.ybuf = reinterpret_cast<double2*>(yb.p);
      a.in = x; a.insel = xsel;
      ev_begin(cls);
      lc(launch_conv_row_fwd(a, stream), "launch_conv_row_fwd");
      lc(launch_conv_col(a, stream), "launch_conv_col");
      a.out = y; a.outsel = ysel;
      a.epi = mode == BLUR_STORE ? SPEC_STORE : mode == BLUR_RESID ? SPEC_RESID : SPEC_AXPY;
      a.g = gg; a.xold = xold; a.xoldsel = xoldsel; a.f = ff; a.tau = tau;
      const int ctas = lc(launch_conv_row_inv(a, stream), "launch_conv_row_inv");
      ev_end();
      launches += 2;
      check_launch();
      return ctas;
    }
    BlurArgs a{};
    a.x = x; a.xsel = xsel; a.y = y; a.ysel = ysel;
    a.w = adjoint ? w_At : w_A;
    a.n1 = n1; a.n2 = n2; a.q1 = q1; a.q2 = q2; a.batch = batch;
    a.bc = bc;
    a.mode = mode; a.g = gg; a.xold = xold; a.xoldsel = xoldsel; a.f = ff; a.tau = tau;
    a.st = stp; a.part = pt;
    int ctas = 0;
    ev_begin(cls);
    launch_blur(a, stream, &ctas);
    ev_end();
    check_launch();
    return ctas;
  }

  // one tensor_map half-pass: col (C = M1 X) or row (C = X M2^T)
  int pass(int kind, bool col, const double* X, int xsel, double* C, int csel, int epi,
           const double* xold, int xoldsel, const double* ff, double tau, const ImgState* stp,
           Partials pt) {
    GemmArgs a{};
    const long long NN = (long long)N;
    if (col) {
      a.A = matrix(kind, 0); a.sA = 0; a.asel = SEL_EXPLICIT;
      a.B = X; a.sB = NN; a.bsel = xsel;
      a.M = n1; a.K = n1; a.N = n2;
    } else {
      a.A = X; a.sA = NN; a.asel = xsel;
      a.B = matrix(kind, 1); a.sB = 0; a.bsel = SEL_EXPLICIT;
      a.M = n1; a.K = n2; a.N = n2;
    }
    a.C = C; a.sC = NN; a.csel = csel;
    a.batch = batch; a.epi = epi; a.d = d; a.dstride = dstride; a.xold = xold; a.xoldsel = xoldsel; a.f = ff;
    a.tau = tau; a.st = stp; a.part = pt; a.img_elems = N;
    int ctas = 0;
    ev_begin(KC_TRANSFORM);
    launch_gemm(a, stream, &ctas);
    ev_end();
    check_launch();
    return ctas;
  }

  // D x = T (d o (T~ x)) (or its first/last halves).  FFT form: T~ rows,
  // [T~ -> d -> T] columns, T rows with the caller's epilogue; dense form: the
  // four GEMM half-passes.  Returns the CTA count of the epilogue launch.
  // D = R^T diag(d) R for the CosineIII algebra (spectral.hpp:147-154):
  // forward R along rows and columns, Hadamard by d, inverse R^T along
  // columns and rows; columns run on transposed images.
  int apply_D_cos(const double* X, int xsel, double* Y, int ysel, int epi_spec, const double* xold,
                  int xoldsel, const double* ff, double tau, const ImgState* stp, Partials pt) {
    if (use_fft_dct()) {
      SpecArgs a = spec_base(stp, pt);
      a.blue2 = dct_tables(1);
      a.in = X; a.insel = xsel; a.out = u.p; a.outsel = SEL_EXPLICIT; a.kind1 = +1; a.epi = SPEC_STORE;
      ev_begin(KC_TRANSFORM);
      lc(launch_dct_rows(a, stream), "launch_dct_rows");
      launch_transpose(u.p, s.p, n1, n2, stream, batch);
      SpecArgs c = a;
      c.n1 = n2; c.n2 = n1;
      c.blue2 = dct_tables(0);
      c.part = Partials{nullptr, 0};
      c.in = s.p; c.out = u.p; c.kind1 = +1; c.epi = SPEC_HADAMARD; c.d = dT.p;
      lc(launch_dct_rows(c, stream), "launch_dct_rows");
      c.in = u.p; c.out = s.p; c.kind1 = -1; c.epi = SPEC_STORE; c.d = nullptr;
      lc(launch_dct_rows(c, stream), "launch_dct_rows");
      launch_transpose(s.p, u.p, n2, n1, stream, batch);
      ev_end();
      launches += 4;
      a.in = u.p; a.insel = SEL_EXPLICIT; a.out = Y; a.outsel = ysel; a.kind1 = -1;
      a.epi = epi_spec; a.xold = xold; a.xoldsel = xoldsel; a.f = ff; a.tau = tau; a.part = pt;
      ev_begin(KC_TRANSFORM);
      const int ctas = lc(launch_dct_rows(a, stream), "launch_dct_rows");
      ev_end();
      check_launch();
      return ctas;
    }
    Partials none{nullptr, 0};
    const int gemm_epi = epi_spec == SPEC_AXPY ? EPI_AXPY : EPI_STORE;
    pass(DBX_KIND_COSINE3, true, X, xsel, u.p, SEL_EXPLICIT, EPI_STORE, nullptr, SEL_EXPLICIT, nullptr, 0, stp, none);
    pass(DBX_KIND_COSINE3, false, u.p, SEL_EXPLICIT, s.p, SEL_EXPLICIT, EPI_HADAMARD, nullptr, SEL_EXPLICIT, nullptr, 0,
         stp, none);
    pass(MK_COSINV, true, s.p, SEL_EXPLICIT, u.p, SEL_EXPLICIT, EPI_STORE, nullptr, SEL_EXPLICIT, nullptr, 0, stp, none);
    return pass(MK_COSINV, false, u.p, SEL_EXPLICIT, Y, ysel, gemm_epi, xold, xoldsel, ff, tau, stp, pt);
  }

  int apply_D(const double* X, int xsel, double* Y, int ysel, int epi_spec, const double* xold,
              int xoldsel, const double* ff, double tau, const ImgState* stp, Partials pt) {
    if (bc == DBX_BC_REFLECTIVE) return apply_D_cos(X, xsel, Y, ysel, epi_spec, xold, xoldsel, ff, tau, stp, pt);
    if (use_fft_dst(false)) {
      SpecArgs a = spec_base(stp, pt);
      a.blue1 = blue_tables(0, false);
      a.blue2 = blue_tables(1, false);
      a.d = d;
      // T~ along rows
      a.in = X; a.insel = xsel; a.out = u.p; a.outsel = SEL_EXPLICIT; a.kind1 = DBX_KIND_ARINV;
      a.epi = SPEC_STORE;
      // transposed stores straight into the column pass's input (no transpose launches)
      // (B1: transposed T~ rows, never the input; B2: the column pass's
      // transposed output, may reuse the consumed input; neither is Y)
      const bool tout = dT.p && dst_tdt_fused() && dst_tout() && Y != s.p && Y != u.p;
      double* B1 = X == s.p ? u.p : s.p;
      double* B2 = B1 == s.p ? u.p : s.p;
      if (tout) {
        a.out = B1;
        a.tout = 1;
      }
      ev_begin(KC_TRANSFORM); lc(launch_dst_rows(a, stream), "launch_dst_rows"); ev_end();
      a.tout = 0;
      // T~ -> d -> T along columns, on the transposed images (columns become
      // contiguous rows: coalesced lines instead of 2-4 column row segments)
      const double* colout = s.p;
      if (tout) {
        SpecArgs c = a;
        c.n1 = n2; c.n2 = n1;
        c.blue2 = blue_tables(0, false);
        c.in = B1; c.out = B2; c.kind1 = DBX_KIND_ARINV; c.kind2 = DBX_KIND_AR; c.epi = SPEC_STORE; c.d = dT.p;
        c.st = stp; c.part = Partials{nullptr, 0};
        c.tout = 1;
        ev_begin(KC_TRANSFORM); lc(launch_dst_rows(c, stream), "launch_dst_rows"); ev_end();
        launches += 1;
        colout = B2;
      } else if (dT.p) {
        ev_begin(KC_TRANSFORM);
        launch_transpose(u.p, s.p, n1, n2, stream, batch);
        SpecArgs c = a;
        c.n1 = n2; c.n2 = n1;
        c.blue2 = blue_tables(0, false);
        c.in = s.p; c.out = u.p; c.kind1 = DBX_KIND_ARINV; c.epi = SPEC_HADAMARD; c.d = dT.p;
        c.st = stp; c.part = Partials{nullptr, 0};
        if (dst_tdt_fused()) {
          // T~, x d^T, T in one row pass (dst_rows kind2)
          c.kind2 = DBX_KIND_AR; c.epi = SPEC_STORE;
          lc(launch_dst_rows(c, stream), "launch_dst_rows");
          launch_transpose(u.p, s.p, n2, n1, stream, batch);
          launches += 3;
          colout = s.p;
        } else {
          lc(launch_dst_rows(c, stream), "launch_dst_rows");
          c.in = u.p; c.out = s.p; c.kind1 = DBX_KIND_AR; c.epi = SPEC_STORE; c.d = nullptr;
          lc(launch_dst_rows(c, stream), "launch_dst_rows");
          launch_transpose(s.p, u.p, n2, n1, stream, batch);
          launches += 4;
          colout = u.p;
        }
        ev_end();
      } else {
        a.in = u.p; a.insel = SEL_EXPLICIT; a.out = s.p; a.outsel = SEL_EXPLICIT;
        a.kind1 = DBX_KIND_ARINV; a.kind2 = DBX_KIND_AR;
        ev_begin(KC_TRANSFORM); lc(launch_dst_cols(a, stream), "launch_dst_cols"); ev_end();
      }
      // T along rows + epilogue
      a.in = colout; a.insel = SEL_EXPLICIT; a.out = Y; a.outsel = ysel; a.kind1 = DBX_KIND_AR; a.kind2 = -1;
      a.epi = epi_spec; a.xold = xold; a.xoldsel = xoldsel; a.f = ff; a.tau = tau;
      ev_begin(KC_TRANSFORM);
      const int ctas = lc(launch_dst_rows(a, stream), "launch_dst_rows");
      ev_end();
      check_launch();
      return ctas;
    }
    Partials none{nullptr, 0};
    const int gemm_epi = epi_spec == SPEC_AXPY ? EPI_AXPY : EPI_STORE;
    pass(DBX_KIND_ARINV, true, X, xsel, u.p, SEL_EXPLICIT, EPI_STORE, nullptr, SEL_EXPLICIT, nullptr, 0, stp, none);
    pass(DBX_KIND_ARINV, false, u.p, SEL_EXPLICIT, s.p, SEL_EXPLICIT, EPI_HADAMARD, nullptr, SEL_EXPLICIT, nullptr, 0, stp, none);
    pass(DBX_KIND_AR, true, s.p, SEL_EXPLICIT, u.p, SEL_EXPLICIT, EPI_STORE, nullptr, SEL_EXPLICIT, nullptr, 0, stp, none);
    return pass(DBX_KIND_AR, false, u.p, SEL_EXPLICIT, Y, ysel, gemm_epi, xold, xoldsel, ff, tau, stp, pt);
  }
};

namespace {

void validate_taps(const double* taps, int q1, int q2) {
  require(taps != nullptr, "Psf: null taps");
  require(q1 >= 0 && q2 >= 0, "Psf: taps must have odd dimensions");
  const size_t n = (size_t)(2 * q1 + 1) * (2 * q2 + 1);
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) {
    require(std::isfinite(taps[i]), "Psf: taps must be finite");
    require(taps[i] >= 0.0, "Psf: taps must be nonnegative");
    s += taps[i];
  }
  require(std::abs(s - 1.0) <= 1e-12, "Psf: taps must sum to 1 (within 1e-12)");
}

// Stage a caller array into the plan (device pointers are used in place).
const double* stage_in(dbx_plan* P, const double* x, DevBuf& buf, size_t count) {
  if (is_device_ptr(x)) return x;
  buf.ensure(count);
  ck(cudaMemcpyAsync(buf.p, x, count * sizeof(double), cudaMemcpyHostToDevice, P->stream), "H2D");
  return buf.p;
}

void stage_out(dbx_plan* P, double* dst, const double* src, size_t count) {
  if (dst == src) return;
  ck(cudaMemcpyAsync(dst, src, count * sizeof(double), cudaMemcpyDefault, P->stream), "D2H");
}

}  // namespace

// ============================================================================
// C++ row-slab D-Landweber (the C5 config): one n x n image split
// into P row slabs of R = n/P rows.  Exchanges are NCCL calls on the plan's
// stream (libnccl.so.2 resolved at run time, so processes that never build a
// communicator do not need it) or, for P in-process ranks on one device, device
// copies / halo views into the neighbour's rows (the parity tests' analogue of
// slab.py's LocalWorld).  Nothing synchronises the host inside the loop: the
// norms are reduced and all-reduced on the device and the bookkeeping runs in
// a one-thread kernel, so every rank takes the same decisions.
// ============================================================================
#include <dlfcn.h>
#include <nccl.h>

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  const char* (*ErrStr)(ncclResult_t) = nullptr;
};

// The NCCL already mapped into the process (torch's) if any, else the system one.
NcclApi& nccl_api() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return a;
    }
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.ErrStr = reinterpret_cast<decltype(a.ErrStr)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.Send && a.Recv && a.GroupStart && a.GroupEnd &&
           a.AllReduce && a.ErrStr;
    if (!a.ok) a.why = "libnccl.so.2 lacks a required symbol";
    return a;
  }();
  return api;
}

void nck(ncclResult_t r, const char* where) {
  if (r != ncclSuccess) throw CudaErr(std::string(where) + ": " + nccl_api().ErrStr(r));
}

}  // namespace

struct dbx_comm {
  ncclComm_t comm = nullptr;
  int nranks = 1, rank = 0;
  bool owned = false;
};

struct dbx_slab {
  int n = 0, P = 1, q = 0, R = 0, C = 0;
  int nloc = 1, rank0 = 0;  // slabs held here: all P (in-process ranks) or this rank's one
  int device = 0;
  bool sep = false;         // separable direct blur (rank-1 mask), else the FFT slab blur
  dbx_comm* comm = nullptr;
  dbx_plan* plan = nullptr; // R x n slab plan: tables, stream, Z^T scratch
  DevBuf x, best, r, s, u, tA, tB, send, recv, top, bot, ext, dTb, part, tot, hist;
  ImgState* st = nullptr;
  double* keep = nullptr;   // dbx_slab_set_iterates: x_k copied here after iteration k (tests)
  int keep_n = 0;
  ~dbx_slab() {
    for (DevBuf* b : {&x, &best, &r, &s, &u, &tA, &tB, &send, &recv, &top, &bot, &ext, &dTb, &part, &tot, &hist})
      b->release();
    if (st) cudaFree(st);
    if (plan) dbx_plan_destroy(plan);
  }
};

// ============================================================================
extern "C" {

const char* dbx_last_error(void) { return g_err.c_str(); }

int dbx_mt19937_64_device(uint64_t seed, uint64_t count, uint64_t* out, int device) {
  std::string e;
  const int st = dbx::mt19937_64_device(seed, count, out, device, e);
  g_err = st ? e : std::string();
  return st;
}

int dbx_gen_honest_device(int rows, int cols, int nshapes, double sinus_amp, uint64_t scene_seed,
                          const double* taps, int q1, int q2, int n1, int n2, double noise_level,
                          uint64_t noise_seed, double* f_true, double* g, int device) {
  std::string e;
  const int st = dbx::gen_honest_device(rows, cols, nshapes, sinus_amp, scene_seed, taps, q1, q2, n1, n2,
                                        noise_level, noise_seed, f_true, g, device, e);
  g_err = st ? e : std::string();
  return st;
}

const char* dbx_version(void) { return "dbx 0.2 sm_100a (FP64 AR stencil / FFT correlation + Bluestein DST-I AR transform)"; }

int dbx_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int ok = 0;
  for (int i = 0; i < n; ++i) {
    cudaDeviceProp pr;
    if (cudaGetDeviceProperties(&pr, i) == cudaSuccess && pr.major == 10) ++ok;
  }
  return ok;
}

int dbx_plan_create(int n1, int n2, int batch, const double* taps, int q1, int q2, int bc,
                    int device, dbx_plan** out) {
  return guarded([&] {
    require(out != nullptr, "dbx_plan_create: null out");
    *out = nullptr;
    require(bc == DBX_BC_ANTIREFLECTIVE || bc == DBX_BC_REFLECTIVE,
            "dbx_plan_create: implemented BCs are AntiReflective and Reflective");
    validate_taps(taps, q1, q2);
    // blur.hpp:26-29 + boundary.hpp:66-81
    require(n1 >= 1 && n2 >= 1, "BlurOperator: empty field of view");
    if (bc == DBX_BC_REFLECTIVE)
      require(q1 <= n1 && q2 <= n2, "reflective support condition violated (q > n)");
    else
      require((q1 == 0 || q1 <= n1 - 2) && (q2 == 0 || q2 <= n2 - 2),
              "anti-reflective support condition violated (q > n-2)");
    require(batch >= 1, "dbx_plan_create: batch must be >= 1");
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
      cudaGetLastError();
      throw CudaErr("no CUDA device: the B200 path has no CPU fallback");
    }
    require(device >= 0 && device < ndev, "dbx_plan_create: bad device index");
    cudaDeviceProp pr;
    ck(cudaGetDeviceProperties(&pr, device), "cudaGetDeviceProperties");
    if (pr.major != 10) throw CudaErr("device is not sm_100 (Blackwell B200)");
    auto P = std::make_unique<dbx_plan>();
    P->n1 = n1; P->n2 = n2; P->batch = batch; P->q1 = q1; P->q2 = q2; P->device = device;
    P->bc = bc;
    P->N = (size_t)n1 * n2;
    const size_t nt = (size_t)(2 * q1 + 1) * (2 * q2 + 1);
    P->taps.assign(taps, taps + nt);
    P->set_dev();
    ck(cudaStreamCreateWithFlags(&P->stream, cudaStreamNonBlocking), "cudaStreamCreate");
    // weights for the correlation form y = sum_t,u w(t,u) P(r-q1+t, c-q2+u):
    // A uses the 180-rotated taps, A' (rotate180 mask, psf.hpp:88-91) the taps.
    std::vector<double> rot(P->taps.rbegin(), P->taps.rend());
    P->w_A = P->upload(rot);
    P->w_At = P->upload(P->taps);
    // symmetrize (psf.hpp:71-85): one orbit average written to four cells
    std::vector<double> s(nt);
    const int W = 2 * q2 + 1;
    auto tp = [&](int i1, int i2) { return P->taps[(size_t)((q1 + i1) * W + (q2 + i2))]; };
    for (int i1 = 0; i1 <= q1; ++i1)
      for (int i2 = 0; i2 <= q2; ++i2) {
        const double avg = (tp(-i1, -i2) + tp(-i1, i2) + tp(i1, -i2) + tp(i1, i2)) / 4.0;
        s[(size_t)((q1 + i1) * W + q2 + i2)] = avg;
        s[(size_t)((q1 - i1) * W + q2 + i2)] = avg;
        s[(size_t)((q1 + i1) * W + q2 - i2)] = avg;
        s[(size_t)((q1 - i1) * W + q2 - i2)] = avg;
      }
    P->sym = P->upload(s);
    ck(cudaMalloc(&P->st, sizeof(ImgState) * (size_t)batch), "cudaMalloc");
    // partial-sum capacity = CTAs per image of the finest launch grid (blur)
    P->part_cap = std::max(((n2 + 63) / 64) * ((n1 + 31) / 32), n1);
    *out = P.release();
  });
}

void dbx_plan_destroy(dbx_plan* plan) {
  if (!plan) return;
  cudaSetDevice(plan->device);
  cudaStreamSynchronize(plan->stream);
  delete plan;
}

void* dbx_plan_stream(dbx_plan* plan) { return plan ? (void*)plan->stream : nullptr; }

int dbx_plan_set_conv(dbx_plan* plan, int conv) {
  return guarded([&] {
    require(plan != nullptr, "null plan");
    require(conv == DBX_CONV_AUTO || conv == DBX_CONV_DIRECT || conv == DBX_CONV_FFT ||
                conv == DBX_CONV_FFT_DENSE,
            "dbx_plan_set_conv: unknown engine");
    plan->conv = conv;
  });
}

int dbx_plan_set_dst(dbx_plan* plan, int engine) {
  return guarded([&] {
    require(plan != nullptr, "null plan");
    require(engine == DBX_DST_AUTO || engine == DBX_DST_DENSE || engine == DBX_DST_FFT ||
                engine == DBX_DST_RADER,
            "dbx_plan_set_dst: unknown engine");
    if (engine != plan->dst)
      for (auto& ax : plan->blue)
        for (auto& B : ax) B.ready = false;  // the DFT core may change: rebuild the tables
    plan->dst = engine;
  });
}

int dbx_plan_set_fusion(dbx_plan* plan, int enable) {
  return guarded([&] {
    require(plan != nullptr, "null plan");
    plan->fusion = enable != 0;
  });
}

int dbx_plan_separable(dbx_plan* plan, int* separable, double* resid) {
  return guarded([&] {
    require(plan != nullptr, "null plan");
    plan->set_dev();
    if (plan->use_fft_conv()) plan->ensure_conv();
    if (separable) *separable = plan->use_fft_conv() && plan->sep_ok && plan->conv != DBX_CONV_FFT_DENSE ? 1 : 0;
    if (resid) *resid = plan->sep_resid;
  });
}

int dbx_plan_engines(dbx_plan* plan, int* conv, int* dst) {
  return guarded([&] {
    require(plan != nullptr, "null plan");
    if (conv) *conv = plan->use_fft_conv() ? DBX_CONV_FFT : DBX_CONV_DIRECT;
    if (dst) *dst = plan->use_fft_dst(false) ? DBX_DST_FFT : DBX_DST_DENSE;
  });
}

#ifdef DBX_PHASES
// Instrumented builds only: read and reset the fused kernels' phase clock sums.
int dbx_debug_phases(unsigned long long* out, int n) { return dbx::fused_debug_phases(out, n); }
#endif

int dbx_plan_pipeline(dbx_plan* plan, int* fused) {
  return guarded([&] {
    require(plan != nullptr, "null plan");
    if (fused) *fused = plan->last_fused;
  });
}

int dbx_plan_set_timing(dbx_plan* plan, int enable) {
  return guarded([&] {
    require(plan != nullptr, "null plan");
    plan->timing = enable != 0;
  });
}

int dbx_plan_kernel_times(dbx_plan* plan, double* ms, int* launches, int max_classes) {
  if (!plan) return 0;
  const int n = std::min(max_classes, (int)KC_NUM);
  for (int i = 0; i < n; ++i) {
    if (ms) ms[i] = plan->kms[i];
    if (launches) launches[i] = plan->kcount[i];
  }
  return KC_NUM;
}

int dbx_plan_kernel_profile(dbx_plan* plan, int idx, char* name, int name_cap, double* ms, int* launches) {
  if (!plan) return 0;
  const int n = (int)plan->kprof.size();
  if (idx >= 0 && idx < n) {
    const auto& e = plan->kprof[(size_t)idx];
    if (name && name_cap > 0) {
      std::strncpy(name, e.first.c_str(), (size_t)name_cap - 1);
      name[name_cap - 1] = 0;
    }
    if (ms) *ms = e.second.first;
    if (launches) *launches = e.second.second;
  }
  return n;
}

int64_t dbx_plan_launch_count(dbx_plan* plan) { return plan ? plan->launches : 0; }

int dbx_blur_apply(dbx_plan* P, const double* x, double* y, int adjoint) {
  return guarded([&] {
    require(P && x && y, "apply: null argument");
    P->set_dev();
    const size_t cnt = P->N * P->batch;
    const double* xin = stage_in(P, x, P->in, cnt);
    double* yout = y;
    if (!is_device_ptr(y)) {
      P->out.ensure(cnt);
      yout = P->out.p;
    }
    P->blur(xin, SEL_EXPLICIT, yout, SEL_EXPLICIT, adjoint != 0, BLUR_STORE, nullptr, nullptr,
            SEL_EXPLICIT, nullptr, 0.0, nullptr, Partials{nullptr, 0}, adjoint ? KC_BLUR_ADJ : KC_BLUR);
    stage_out(P, y, yout, cnt);
    ck(cudaStreamSynchronize(P->stream), "sync");
  });
}

int dbx_precond_build(dbx_plan* P, double alpha) {
  return guarded([&] {
    require(P != nullptr, "null plan");
    require(alpha >= 0.0, "tikhonov_filter: alpha must be nonnegative");
    // eig_antireflective preconditions (spectral.hpp:122-126); eig_reflective
    // has none beyond the (symmetrised) mask's symmetry (spectral.hpp:75-84)
    if (P->bc == DBX_BC_ANTIREFLECTIVE) {
      require(P->n1 >= 3 && P->n2 >= 3, "eig_antireflective: sizes must be >= 3");
      require(P->q1 <= P->n1 - 2 && P->q2 <= P->n2 - 2, "eig_antireflective: support condition violated");
    }
    P->set_dev();
    P->ensure_d(P->N);
    P->dstride = 0;
    int* flag = nullptr;
    ck(cudaMalloc(&flag, sizeof(int)), "cudaMalloc");
    ck(cudaMemsetAsync(flag, 0, sizeof(int), P->stream), "memset");
    launch_build_filter(P->sym, P->q1, P->q2, P->n1, P->n2, alpha, P->d, flag, P->stream,
                        P->bc == DBX_BC_REFLECTIVE ? 1 : 0);
    P->launches += 3;
    P->check_launch();
    int hflag = 0;
    ck(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, P->stream), "D2H");
    ck(cudaStreamSynchronize(P->stream), "sync");
    cudaFree(flag);
    P->have_d = false;
    require(alpha > 0.0 || hflag == 0, "tikhonov_filter: alpha = 0 with a zero eigenvalue");
    P->have_d = true;
    P->dT.ensure(P->N);
    launch_transpose(P->d, P->dT.p, P->n1, P->n2, P->stream);
    ck(cudaStreamSynchronize(P->stream), "transpose");
  });
}

// ---------------------------------------------------------------------------
// Row-slab building blocks (C5 multi-GPU decomposition, slab.py).  The plan is
// created for ONE slab (n1 = slab rows, n2 = full width, batch 1); all
// pointers are device pointers; the caller supplies halos / transposes.
// ---------------------------------------------------------------------------
static void sum_partials(dbx_plan* P, int slot, int cnt, double* out) {
  std::vector<double> h((size_t)cnt);
  ck(cudaMemcpyAsync(h.data(), P->part.p + (size_t)slot * P->part_cap, cnt * sizeof(double),
                     cudaMemcpyDeviceToHost, P->stream), "D2H");
  ck(cudaStreamSynchronize(P->stream), "sync");
  double acc = 0.0;
  for (double v : h) acc += v;  // fixed order
  *out = acc;
}

int dbx_slab_blur(dbx_plan* P, const double* x_ext, double* y, int adjoint, const double* g, double* norm2) {
  return guarded([&] {
    require(P && x_ext && y, "slab_blur: null argument");
    require(P->batch == 1, "slab_blur: one slab per plan");
    require(is_device_ptr(x_ext) && is_device_ptr(y) && (!g || is_device_ptr(g)), "slab_blur: device pointers");
    require(P->use_fft_conv(), "slab_blur: needs the FFT correlation engine");
    require(P->bc == DBX_BC_ANTIREFLECTIVE, "slab_blur: anti-reflective slabs only");
    P->set_dev();
    P->ensure_conv();
    P->zb.ensure((size_t)(P->n1 + 2 * P->q1) * P->Lh * 2);
    P->part.ensure((size_t)NUM_SLOTS * P->part_cap);
    Partials pt{P->part.p, P->part_cap};
    SpecArgs a = P->spec_base(nullptr, pt);
    a.conv.tw1 = reinterpret_cast<const double2*>(P->tw1);
    a.conv.tw2 = reinterpret_cast<const double2*>(P->tw2);
    P->set_kernel(a.conv, adjoint);
    a.conv.L1 = P->L1; a.conv.L2 = P->L2; a.conv.Lh = P->Lh;
    a.zbuf = reinterpret_cast<double2*>(P->zb.p);
    a.ybuf = reinterpret_cast<double2*>(P->yb.p);
    // rows of the caller-extended slab (halo rows / global AR rows included)
    a.in = x_ext;
    a.n1 = P->n1 + 2 * P->q1;
    lc(launch_conv_row_fwd(a, P->stream), "launch_conv_row_fwd");
    a.n1 = P->n1;
    a.preext = 1;
    lc(launch_conv_col(a, P->stream), "launch_conv_col");
    a.preext = 0;
    a.out = y;
    a.epi = g ? SPEC_RESID : SPEC_STORE;
    a.g = g;
    const int ctas = lc(launch_conv_row_inv(a, P->stream), "launch_conv_row_inv");
    P->launches += 3;
    P->check_launch();
    if (g && norm2) sum_partials(P, SLOT_R2, ctas, norm2);
    ck(cudaStreamSynchronize(P->stream), "sync");
  });
}

int dbx_slab_rows(dbx_plan* P, int kind, const double* x, double* y, int epi, const double* aux, const double* f,
                  double tau, double* norms2) {
  return guarded([&] {
    require(P && x && y, "slab_rows: null argument");
    require(P->batch == 1, "slab_rows: one slab per plan");
    require(kind == DBX_KIND_SINEI || kind == DBX_KIND_AR || kind == DBX_KIND_ARINV, "slab_rows: unsupported kind");
    require(epi == DBX_SLAB_STORE || epi == DBX_SLAB_HADAMARD || epi == DBX_SLAB_AXPY, "slab_rows: unknown epilogue");
    require(epi == DBX_SLAB_STORE || aux != nullptr, "slab_rows: missing operand");
    require(is_device_ptr(x) && is_device_ptr(y), "slab_rows: device pointers");
    const bool sine = kind == DBX_KIND_SINEI;
    require(P->use_fft_dst(sine), "slab_rows: needs the FFT-form DST");
    P->set_dev();
    P->part.ensure((size_t)NUM_SLOTS * P->part_cap);
    Partials pt{P->part.p, P->part_cap};
    SpecArgs a = P->spec_base(nullptr, pt);
    a.blue2 = P->blue_tables(1, sine);
    a.in = x;
    a.out = y;
    a.kind1 = kind;
    a.kind2 = -1;
    a.epi = epi == DBX_SLAB_STORE ? SPEC_STORE : epi == DBX_SLAB_HADAMARD ? SPEC_HADAMARD : SPEC_AXPY;
    a.d = epi == DBX_SLAB_HADAMARD ? aux : nullptr;
    a.xold = epi == DBX_SLAB_AXPY ? aux : nullptr;
    a.f = epi == DBX_SLAB_AXPY ? f : nullptr;
    a.tau = tau;
    const int ctas = lc(launch_dst_rows(a, P->stream), "launch_dst_rows");
    ++P->launches;
    P->check_launch();
    if (epi == DBX_SLAB_AXPY && norms2) {
      sum_partials(P, SLOT_X2, ctas, norms2);
      if (f) sum_partials(P, SLOT_XF2, ctas, norms2 + 1);
      else norms2[1] = 0.0;
    }
    ck(cudaStreamSynchronize(P->stream), "sync");
  });
}

int dbx_precond_block(dbx_plan* P, int n1g, int n2g, double alpha, int r0, int nr, int c0, int nc, int transpose,
                      double* out) {
  return guarded([&] {
    require(P && out, "precond_block: null argument");
    require(alpha >= 0.0, "tikhonov_filter: alpha must be nonnegative");
    require(n1g >= 3 && n2g >= 3 && P->q1 <= n1g - 2 && P->q2 <= n2g - 2, "eig_antireflective: support condition");
    require(r0 >= 0 && nr > 0 && r0 + nr <= n1g && c0 >= 0 && nc > 0 && c0 + nc <= n2g, "precond_block: block");
    require(is_device_ptr(out), "precond_block: device pointer");
    P->set_dev();
    int* flag = nullptr;
    ck(cudaMalloc(&flag, sizeof(int)), "cudaMalloc");
    ck(cudaMemsetAsync(flag, 0, sizeof(int), P->stream), "memset");
    launch_build_filter_block(P->sym, P->q1, P->q2, n1g, n2g, alpha, r0, nr, c0, nc, transpose != 0, out, flag,
                              P->stream, P->bc == DBX_BC_REFLECTIVE ? 1 : 0);
    P->launches += 3;
    P->check_launch();
    int hflag = 0;
    ck(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, P->stream), "D2H");
    ck(cudaStreamSynchronize(P->stream), "sync");
    cudaFree(flag);
    require(alpha > 0.0 || hflag == 0, "tikhonov_filter: alpha = 0 with a zero eigenvalue");
  });
}

int dbx_slab_extend(dbx_plan* P, const double* x, const double* top, const double* bot, double* x_ext) {
  return guarded([&] {
    require(P && x && x_ext, "slab_extend: null argument");
    require(is_device_ptr(x) && is_device_ptr(x_ext) && (!top || is_device_ptr(top)) && (!bot || is_device_ptr(bot)),
            "slab_extend: device pointers");
    require(P->n1 >= P->q1 + 1, "slab_extend: slab must hold at least q1 + 1 rows");
    P->set_dev();
    const size_t row = (size_t)P->n2 * sizeof(double), q = (size_t)P->q1;
    cudaStream_t s = P->stream;
    ck(cudaMemcpyAsync(x_ext + q * P->n2, x, row * P->n1, cudaMemcpyDeviceToDevice, s), "copy");
    if (top) ck(cudaMemcpyAsync(x_ext, top, row * q, cudaMemcpyDeviceToDevice, s), "copy");
    if (bot) ck(cudaMemcpyAsync(x_ext + (q + P->n1) * P->n2, bot, row * q, cudaMemcpyDeviceToDevice, s), "copy");
    launch_slab_ar_rows(x, x_ext, P->n1, P->n2, P->q1, top == nullptr, bot == nullptr, s);
    ++P->launches;
    P->check_launch();
    ck(cudaStreamSynchronize(s), "sync");
  });
}

int dbx_slab_pack(dbx_plan* P, const double* x, double* blocks, int parts, int unpack) {
  return guarded([&] {
    require(P && x && blocks && parts > 0 && P->n2 % parts == 0, "slab_pack: bad argument");
    require(is_device_ptr(x) && is_device_ptr(blocks), "slab_pack: device pointers");
    P->set_dev();
    const size_t cb = (size_t)P->n2 / parts, w = cb * sizeof(double), pitch = (size_t)P->n2 * sizeof(double);
    for (int p = 0; p < parts; ++p) {
      double* blk = blocks + (size_t)p * P->n1 * cb;
      const double* col = x + (size_t)p * cb;
      if (unpack)
        ck(cudaMemcpy2DAsync(const_cast<double*>(col), pitch, blk, w, w, P->n1, cudaMemcpyDeviceToDevice, P->stream),
           "unpack");
      else
        ck(cudaMemcpy2DAsync(blk, w, col, pitch, w, P->n1, cudaMemcpyDeviceToDevice, P->stream), "pack");
    }
    ck(cudaStreamSynchronize(P->stream), "sync");
  });
}

int dbx_transpose(dbx_plan* P, const double* in, double* out, int rows, int cols) {
  return guarded([&] {
    require(P && in && out && rows > 0 && cols > 0, "transpose: bad argument");
    require(is_device_ptr(in) && is_device_ptr(out), "transpose: device pointers");
    P->set_dev();
    launch_transpose(in, out, rows, cols, P->stream);
    ++P->launches;
    P->check_launch();
    ck(cudaStreamSynchronize(P->stream), "sync");
  });
}

int dbx_precond_build_sweep(dbx_plan* P, const double* alphas) {
  return guarded([&] {
    require(P && alphas, "null argument");
    if (P->bc == DBX_BC_ANTIREFLECTIVE) {
      require(P->n1 >= 3 && P->n2 >= 3, "eig_antireflective: sizes must be >= 3");
      require(P->q1 <= P->n1 - 2 && P->q2 <= P->n2 - 2, "eig_antireflective: support condition violated");
    }
    for (int b = 0; b < P->batch; ++b) require(alphas[b] >= 0.0, "tikhonov_filter: alpha must be nonnegative");
    P->set_dev();
    const size_t B = (size_t)P->batch;
    P->ensure_d(B * P->N);
    int* flag = nullptr;
    ck(cudaMalloc(&flag, B * sizeof(int)), "cudaMalloc");
    ck(cudaMemsetAsync(flag, 0, B * sizeof(int), P->stream), "memset");
    for (size_t b = 0; b < B; ++b)
      launch_build_filter(P->sym, P->q1, P->q2, P->n1, P->n2, alphas[b], P->d + b * P->N, flag + b, P->stream,
                          P->bc == DBX_BC_REFLECTIVE ? 1 : 0);
    P->launches += 3 * (int64_t)B;
    P->check_launch();
    std::vector<int> hflag(B);
    ck(cudaMemcpyAsync(hflag.data(), flag, B * sizeof(int), cudaMemcpyDeviceToHost, P->stream), "D2H");
    ck(cudaStreamSynchronize(P->stream), "sync");
    cudaFree(flag);
    P->have_d = false;
    for (size_t b = 0; b < B; ++b)
      require(alphas[b] > 0.0 || hflag[b] == 0, "tikhonov_filter: alpha = 0 with a zero eigenvalue");
    P->have_d = true;
    P->dstride = P->N;
    P->dT.ensure(B * P->N);
    launch_transpose(P->d, P->dT.p, P->n1, P->n2, P->stream, (int)B);
    ck(cudaStreamSynchronize(P->stream), "transpose");
  });
}

int dbx_precond_eigs(dbx_plan* P, double* d_out) {
  return guarded([&] {
    require(P && d_out, "null argument");
    require(P->have_d, "precondition: filter not built");
    P->set_dev();
    stage_out(P, d_out, P->d, P->N);
    ck(cudaStreamSynchronize(P->stream), "sync");
  });
}

int dbx_precond_set_eigs(dbx_plan* P, const double* dd) {
  return guarded([&] {
    require(P && dd, "null argument");
    P->set_dev();
    P->ensure_d(P->N);
    P->dstride = 0;
    ck(cudaMemcpyAsync(P->d, dd, P->N * sizeof(double), cudaMemcpyDefault, P->stream), "copy");
    ck(cudaStreamSynchronize(P->stream), "sync");
    P->have_d = true;
    P->dT.ensure(P->N);
    launch_transpose(P->d, P->dT.p, P->n1, P->n2, P->stream);
    ck(cudaStreamSynchronize(P->stream), "transpose");
  });
}

int dbx_precond_apply(dbx_plan* P, const double* r, double* y) {
  return guarded([&] {
    require(P && r && y, "null argument");
    require(P->have_d, "precondition_apply: filter not built");
    require(P->bc == DBX_BC_REFLECTIVE || (P->n1 >= 3 && P->n2 >= 3),
            "tensor_apply: anti-reflective transform needs sizes >= 3");
    P->set_dev();
    const size_t cnt = P->N * P->batch;
    const double* rin = stage_in(P, r, P->in, cnt);
    P->u.ensure(cnt);
    P->s.ensure(cnt);
    double* yout = y;
    if (!is_device_ptr(y)) {
      P->out.ensure(cnt);
      yout = P->out.p;
    }
    P->apply_D(rin, SEL_EXPLICIT, yout, SEL_EXPLICIT, SPEC_STORE, nullptr, SEL_EXPLICIT, nullptr, 0.0,
               nullptr, Partials{nullptr, 0});
    stage_out(P, y, yout, cnt);
    ck(cudaStreamSynchronize(P->stream), "sync");
  });
}

int dbx_tensor_apply(dbx_plan* P, int kind, const double* x, double* y) {
  return guarded([&] {
    require(P && x && y, "null argument");
    require(kind == DBX_KIND_SINEI || kind == DBX_KIND_AR || kind == DBX_KIND_ARINV || kind == DBX_KIND_COSINE3,
            "tensor_apply: unsupported kind");
    if (kind == DBX_KIND_AR || kind == DBX_KIND_ARINV)
      require(P->n1 >= 3 && P->n2 >= 3, "tensor_apply: anti-reflective transform needs sizes >= 3");
    P->set_dev();
    const size_t cnt = P->N * P->batch;
    const double* xin = stage_in(P, x, P->in, cnt);
    P->u.ensure(cnt);
    double* yout = y;
    if (!is_device_ptr(y)) {
      P->out.ensure(cnt);
      yout = P->out.p;
    }
    Partials none{nullptr, 0};
    const bool sine = kind == DBX_KIND_SINEI;
    if (kind == DBX_KIND_COSINE3) {
      // R along rows, then (transposed) along columns (transforms.hpp:198-204)
      if (P->use_fft_dct()) {
        P->s.ensure(cnt);
        SpecArgs a = P->spec_base(nullptr, none);
        a.blue2 = P->dct_tables(1);
        a.in = xin; a.out = P->u.p; a.kind1 = +1; a.epi = SPEC_STORE;
        P->ev_begin(KC_TRANSFORM);
        lc(launch_dct_rows(a, P->stream), "launch_dct_rows");
        launch_transpose(P->u.p, P->s.p, P->n1, P->n2, P->stream, P->batch);
        SpecArgs c = a;
        c.n1 = P->n2; c.n2 = P->n1; c.blue2 = P->dct_tables(0);
        c.in = P->s.p; c.out = P->u.p;
        lc(launch_dct_rows(c, P->stream), "launch_dct_rows");
        launch_transpose(P->u.p, yout, P->n2, P->n1, P->stream, P->batch);
        P->ev_end();
        P->launches += 3;
        P->check_launch();
      } else {
        P->pass(DBX_KIND_COSINE3, true, xin, SEL_EXPLICIT, P->u.p, SEL_EXPLICIT, EPI_STORE, nullptr, SEL_EXPLICIT,
                nullptr, 0, nullptr, none);
        P->pass(DBX_KIND_COSINE3, false, P->u.p, SEL_EXPLICIT, yout, SEL_EXPLICIT, EPI_STORE, nullptr, SEL_EXPLICIT,
                nullptr, 0, nullptr, none);
      }
    } else if (P->use_fft_dst(sine)) {
      // rows then columns (Kronecker order is immaterial; the reference runs
      // columns first, transforms.hpp:183-190)
      SpecArgs a = P->spec_base(nullptr, none);
      a.blue1 = P->blue_tables(0, sine);
      a.blue2 = P->blue_tables(1, sine);
      a.in = xin; a.out = P->u.p; a.kind1 = kind; a.kind2 = -1; a.epi = SPEC_STORE;
      P->ev_begin(KC_TRANSFORM); lc(launch_dst_rows(a, P->stream), "launch_dst_rows"); P->ev_end();
      a.in = P->u.p; a.out = yout;
      P->ev_begin(KC_TRANSFORM); lc(launch_dst_cols(a, P->stream), "launch_dst_cols"); P->ev_end();
      P->check_launch();
    } else {
      P->pass(kind, true, xin, SEL_EXPLICIT, P->u.p, SEL_EXPLICIT, EPI_STORE, nullptr, SEL_EXPLICIT, nullptr, 0, nullptr, none);
      P->pass(kind, false, P->u.p, SEL_EXPLICIT, yout, SEL_EXPLICIT, EPI_STORE, nullptr, SEL_EXPLICIT, nullptr, 0, nullptr, none);
    }
    stage_out(P, y, yout, cnt);
    ck(cudaStreamSynchronize(P->stream), "sync");
  });
}

static int run_impl(dbx_plan* P, const double* g, const double* f_true, double tau, int max_iters, int stop_kind,
                    int fixed_iters, double resid_eps, int use_precond, double* restored, double* rre_hist,
                    double* res_hist, int* best_iter, int* iters_done, double* x_hist, int method,
                    int img_base = 0);

int dbx_landweber_run(dbx_plan* P, const double* g, const double* f_true, double tau,
                      int max_iters, int stop_kind, int fixed_iters, double resid_eps,
                      int use_precond, double* restored, double* rre_hist, double* res_hist,
                      int* best_iter, int* iters_done, double* x_hist) {
  return run_impl(P, g, f_true, tau, max_iters, stop_kind, fixed_iters, resid_eps, use_precond, restored, rre_hist,
                  res_hist, best_iter, iters_done, x_hist, 0);
}

int dbx_cgls_run(dbx_plan* P, const double* g, const double* f_true, int max_iters, int stop_kind, int fixed_iters,
                 double resid_eps, int use_precond, double* restored, double* rre_hist, double* res_hist,
                 int* best_iter, int* iters_done, double* x_hist) {
  return run_impl(P, g, f_true, 1.0, max_iters, stop_kind, fixed_iters, resid_eps, use_precond, restored, rre_hist,
                  res_hist, best_iter, iters_done, x_hist, 1);
}

static int run_impl(dbx_plan* P, const double* g, const double* f_true, double tau, int max_iters, int stop_kind,
                    int fixed_iters, double resid_eps, int use_precond, double* restored, double* rre_hist,
                    double* res_hist, int* best_iter, int* iters_done, double* x_hist, int method,
                    int img_base) {
  return guarded([&] {
    require(P && g && restored, "landweber: null argument");
    // solver.hpp:66-72, 17-32
    require(tau > 0.0, "landweber: tau must be positive");
    require(max_iters >= 1, "landweber: max_iters must be at least 1");
    require(stop_kind >= 0 && stop_kind <= 2, "landweber: unknown stopping rule");
    require(stop_kind != DBX_STOP_FIXED || fixed_iters >= 0, "StoppingRule: negative iteration count");
    require(stop_kind != DBX_STOP_RESIDUAL || resid_eps > 0.0, "StoppingRule: threshold must be positive");
    if (use_precond) {
      require(P->have_d, "d_landweber: preconditioner not built");
      require(P->bc == DBX_BC_REFLECTIVE || (P->n1 >= 3 && P->n2 >= 3),
              "tensor_apply: anti-reflective transform needs sizes >= 3");
    }
    P->set_dev();
    const int B = P->batch;
    const size_t N = P->N, cnt = N * B;
    const int total = stop_kind == DBX_STOP_FIXED ? fixed_iters : max_iters;
    const bool track = f_true != nullptr;
    cudaStream_t s = P->stream;

    // ---- stage inputs (H2D for host arrays) ----
    const double* gd = stage_in(P, g, P->g, cnt);
    const double* fd = track ? stage_in(P, f_true, P->f, cnt) : nullptr;
    P->r.ensure(cnt);
    P->s.ensure(cnt);
    if (use_precond) P->u.ensure(cnt);
    P->X3.ensure(3 * cnt);
    P->part.ensure((size_t)B * NUM_SLOTS * P->part_cap);
    const int H = std::max(total, 1);
    P->rre.ensure((size_t)B * H);
    P->res.ensure((size_t)B * H);
    const bool want_xh = x_hist != nullptr;
    if (want_xh) P->xh.ensure((size_t)H * cnt);
    Partials pt{P->part.p, P->part_cap};

    launch_state_init(P->st, B, s);
    P->fincnt.ensure((size_t)B);
    ck(cudaMemsetAsync(P->fincnt.p, 0, (size_t)B * sizeof(unsigned), s), "memset");
    launch_norms_init(gd, fd, B, N, P->st, pt, s);
    P->launches += 3;
    // x_0 = 0 in buffer 0, r_0 = g
    ck(cudaMemsetAsync(P->X3.p, 0, cnt * sizeof(double), s), "memset");
    ck(cudaMemcpyAsync(P->r.p, gd, cnt * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
    P->check_launch();

    // Fused FFT-form pipeline (fused.cu): 6 launches + finalize per iteration.
    P->prepare(use_precond != 0);
    const bool fused = method == 0 && use_precond && P->bc == DBX_BC_ANTIREFLECTIVE && P->n1 == P->n2 &&
                       P->use_fft_conv() && P->use_fft_dst(false) &&
                       P->fusion &&
                       P->blue_tables(1, false).core != CORE_RADER &&
                       fused_supported(P->L2, P->blue_tables(1, false).M,
                                       P->blue_tables(1, false).core == CORE_BLUE);
    // Separable fused pipeline (rank-1 mask): direct row passes in the row
    // kernels and a real column pass instead of the row FFTs and the complex
    // column pass (DBX_NO_SEP_ROWS=1 keeps the FFT rows, diagnostic A/B)
    static const bool no_sep_rows = [] {
      const char* e = std::getenv("DBX_NO_SEP_ROWS");
      return e && e[0] == '1';
    }();
    const bool sepd = fused && !no_sep_rows && P->sep_ok && P->conv != DBX_CONV_FFT_DENSE &&
                      conv_sep_supported(P->q1) &&
                      fused_sep_supported(P->L2, P->blue_tables(1, false).M,
                                          P->blue_tables(1, false).core == CORE_BLUE, P->n2, P->q2);
    P->last_fused = fused ? (sepd ? 2 : 1) : 0;
    SpecArgs fa0 = P->spec_base(P->st, pt);
    if (fused) {
      fa0.conv.tw1 = reinterpret_cast<const double2*>(P->tw1);
      fa0.conv.tw2 = reinterpret_cast<const double2*>(P->tw2);
      fa0.conv.L1 = P->L1; fa0.conv.L2 = P->L2; fa0.conv.Lh = P->Lh;
      fa0.zbuf = reinterpret_cast<double2*>(P->zb.p);
      fa0.ybuf = reinterpret_cast<double2*>(P->yb.p);
      fa0.blue1 = P->blue_tables(0, false);
      fa0.blue2 = P->blue_tables(1, false);
      fa0.d = P->d;
      fa0.g = gd;
      fa0.f = fd;
      fa0.tau = tau;
      fa0.ztrans = 1;
      fa0.dT = P->dT.p;
    }
    // ---- reblurred (preconditioned) CGLS state (cg.cu) ----
    if (method == 1) {
      for (DevBuf* b : {&P->cg_p, &P->cg_q, &P->cg_s, &P->cg_z, &P->cg_zero}) b->ensure(cnt);
      P->cg_part.ensure((size_t)B * P->part_cap);
      P->cg_sc.ensure((size_t)B * 4);
      ck(cudaMemsetAsync(P->cg_zero.p, 0, cnt * sizeof(double), s), "memset");
    }
    CgScalars* cgs = method == 1 ? reinterpret_cast<CgScalars*>(P->cg_sc.p) : nullptr;
    auto cg_precond = [&](const double* in, double* out) -> const double* {
      if (!use_precond) return in;  // plain CGLS: z = s
      P->apply_D(in, SEL_EXPLICIT, out, SEL_EXPLICIT, SPEC_STORE, nullptr, SEL_EXPLICIT, nullptr, 0.0, P->st,
                 Partials{nullptr, 0});
      return out;
    };
    auto cg_direction = [&](int init) {  // s = A' r, z = D s, gamma = <s, z>, p = z + beta p
      P->blur(P->r.p, SEL_EXPLICIT, P->cg_s.p, SEL_EXPLICIT, true, BLUR_STORE, nullptr, nullptr, SEL_EXPLICIT,
              nullptr, 0.0, P->st, pt, KC_BLUR_ADJ);
      const double* z = cg_precond(P->cg_s.p, P->cg_z.p);
      const int cnt_d = launch_cg_dot(P->st, P->cg_s.p, z, B, N, P->cg_part.p, P->part_cap, s);
      launch_cg_beta(P->st, cgs, P->cg_part.p, P->part_cap, cnt_d, init, B, s);
      if (init) ck(cudaMemcpyAsync(P->cg_p.p, z, cnt * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
      else launch_cg_xpay(P->st, cgs, z, P->cg_p.p, B, N, s);
      P->launches += 3;
      P->check_launch();
    };
    auto enqueue_pre = [&]() {
      if (method == 1) {
        cg_direction(1);
        return;
      }
      if (!fused) return;
      if (sepd) {
        // row pass of A' r_0 = A' g (r = g: no A x rows yet)
        SpecArgs a = fa0;
        P->set_kernel(a.conv, true);
        a.in = nullptr; a.insel = SEL_EXPLICIT;
        P->ev_begin(KC_BLUR_ADJ);
        lc(launch_fused(FUSED_RESID_SEP, a, s), "rows_resid_sep");
        P->ev_end();
        return;
      }
      // spectrum of the AR-extended r_0 = g for the first A' apply
      SpecArgs a = fa0;
      a.in = gd; a.insel = SEL_EXPLICIT;
      P->ev_begin(KC_BLUR_ADJ);
      lc(launch_conv_row_fwd(a, s), "launch_conv_row_fwd");
      P->ev_end();
    };
    // DBX_FIN_FUSED=1: the fused pipelines run the iteration's finalize as the
    // last-block tail of their residual kernel (finalize.cuh; one launch fewer
    // per iteration).  Measured slower on every config (C1 1595 vs 1623, C2
    // 3982 vs 4018, C3 25430 vs 25545 Mpx-it/s, profiles/r02_fin_fused_ab.txt):
    // the fence + atomic + one CTA's serial tail cost more than a graph
    // kernel boundary.  Off by default; parity-tested on.
    static const bool fin_fused = [] { const char* e = getenv("DBX_FIN_FUSED"); return e && e[0] == '1'; }();
    auto make_fa = [&](int k, int cnt_x, int cnt_r) {
      FinalizeArgs fa{};
      fa.st = P->st; fa.part = pt; fa.cnt_x = cnt_x; fa.cnt_r = cnt_r; fa.k = k;
      fa.hist_len = H; fa.rre_hist = P->rre.p; fa.res_hist = P->res.p;
      fa.track = track ? 1 : 0; fa.stop_kind = stop_kind; fa.resid_eps = resid_eps; fa.batch = B;
      return fa;
    };
    auto set_fin = [&](SpecArgs& a, int k, int cnt_x) {
      if (!fin_fused) return;
      a.fin = make_fa(k, cnt_x, -1);
      a.fin_cnt = reinterpret_cast<unsigned*>(P->fincnt.p);
    };
    auto enqueue_fused_sep = [&](int k) {
      SpecArgs a = fa0;
      double* Yr = reinterpret_cast<double*>(P->yb.p);
      // K1: column pass of A' (real): Z'^T -> Y' = A' r (row-major)
      P->set_kernel(a.conv, true);
      P->ev_begin(KC_BLUR_ADJ); lc(launch_cols_sep_real(a, s), "cols_sep_real"); P->ev_end();
      // K2: s = A' r rows -> T~ along rows -> u
      a.out = P->u.p; a.outsel = SEL_EXPLICIT;
      P->ev_begin(KC_TRANSFORM); lc(launch_fused(FUSED_TT_SEP, a, s), "rows_tt_sep"); P->ev_end();
      // K3: columns of u: T~ -> d -> T, into row-major s
      a.in = P->u.p; a.insel = SEL_EXPLICIT; a.out = P->s.p; a.outsel = SEL_EXPLICIT;
      a.kind1 = DBX_KIND_ARINV; a.kind2 = DBX_KIND_AR; a.epi = SPEC_STORE;
      P->ev_begin(KC_TRANSFORM); lc(launch_fused(FUSED_DST_TCOLS, a, s), "dst_tcols"); P->ev_end();
      // K4: T along rows -> x_k -> norms -> row pass of A x_k -> Z^T
      P->set_kernel(a.conv, false);
      a.in = P->s.p; a.out = P->X3.p; a.outsel = SEL_NXT; a.xold = P->X3.p; a.xoldsel = SEL_CUR;
      P->ev_begin(KC_TRANSFORM);
      const int cnt_x = lc(launch_fused(FUSED_T_AXPY_SEP, a, s), "rows_t_axpy_sep");
      P->ev_end();
      // K5: column pass of A (real): Z^T -> Y = A x_k
      P->ev_begin(KC_BLUR); lc(launch_cols_sep_real(a, s), "cols_sep_real"); P->ev_end();
      // K6: r = g - A x_k + ||r||^2 -> row pass of A' r -> Z'^T
      P->set_kernel(a.conv, true);
      a.in = Yr; a.insel = SEL_EXPLICIT;
      set_fin(a, k, cnt_x);
      P->ev_begin(KC_BLUR);
      const int cnt_r = lc(launch_fused(FUSED_RESID_SEP, a, s), "rows_resid_sep");
      P->ev_end();
      return std::make_pair(cnt_x, cnt_r);
    };
    auto enqueue_fused = [&](int k) {
      if (sepd) return enqueue_fused_sep(k);
      SpecArgs a = fa0;
      // K1: column pass of A' (spectral AR extension, kernel spectrum of the rotated mask)
      P->set_kernel(a.conv, true);
      P->ev_begin(KC_BLUR_ADJ); lc(launch_conv_col(a, s), "launch_conv_col"); P->ev_end();
      // K2: inverse row FFT -> A'r rows -> T~ along rows -> u
      a.out = P->u.p; a.outsel = SEL_EXPLICIT;
      P->ev_begin(KC_TRANSFORM); lc(launch_fused(FUSED_AINV_TT, a, s), "rows_ainv_tt"); P->ev_end();
      // K3: columns of u (= rows of u^T, contiguous): T~ -> d -> T, into row-major s
      a.in = P->u.p; a.insel = SEL_EXPLICIT; a.out = P->s.p; a.outsel = SEL_EXPLICIT;
      a.kind1 = DBX_KIND_ARINV; a.kind2 = DBX_KIND_AR; a.epi = SPEC_STORE;
      P->ev_begin(KC_TRANSFORM); lc(launch_fused(FUSED_DST_TCOLS, a, s), "dst_tcols"); P->ev_end();
      // K4: T along rows -> x_k = x_{k-1} + tau (.) + norms -> forward row FFT for A x_k
      a.in = P->s.p; a.out = P->X3.p; a.outsel = SEL_NXT; a.xold = P->X3.p; a.xoldsel = SEL_CUR;
      P->ev_begin(KC_TRANSFORM);
      const int cnt_x = lc(launch_fused(FUSED_T_AXPY_AFWD, a, s), "rows_t_axpy_afwd");
      P->ev_end();
      // K5: column pass of A
      P->set_kernel(a.conv, false);
      P->ev_begin(KC_BLUR); lc(launch_conv_col(a, s), "launch_conv_col"); P->ev_end();
      // K6: inverse row FFT -> r_k = g - A x_k + ||r||^2 -> forward row FFT for the next A'
      set_fin(a, k, cnt_x);
      P->ev_begin(KC_BLUR);
      const int cnt_r = lc(launch_fused(FUSED_AINV_RESID, a, s), "rows_ainv_resid");
      P->ev_end();
      return std::make_pair(cnt_x, cnt_r);
    };

    auto enqueue = [&](int k) {
      int cnt_x = 0;
      if (fused) {
        const auto cr = enqueue_fused(k);
        if (!fin_fused) {
          const FinalizeArgs fa = make_fa(k, cr.first, cr.second);
          P->ev_begin(KC_FINALIZE);
          launch_finalize(fa, s);
          P->ev_end();
        }
        P->check_launch();
        if (want_xh) {
          launch_select_copy(P->X3.p, P->st, 0, B, N, P->xh.p + (size_t)(k - 1) * cnt, s);
          ++P->launches;
        }
        return;
      }
      if (method == 1) {
        // q' = 0 - A p (||q||^2 in the residual slot) -> alpha -> x, r updates
        const int cnt_q = P->blur(P->cg_p.p, SEL_EXPLICIT, P->cg_q.p, SEL_EXPLICIT, false, BLUR_RESID,
                                  P->cg_zero.p, nullptr, SEL_EXPLICIT, nullptr, 0.0, P->st, pt, KC_BLUR);
        launch_cg_alpha(P->st, cgs, pt, cnt_q, B, s);
        const int cnt_u = launch_cg_update(P->X3.p, P->st, cgs, P->cg_p.p, P->cg_q.p, P->r.p, fd, B, N, pt, s);
        P->launches += 2;
        FinalizeArgs fa{};
        fa.st = P->st; fa.part = pt; fa.cnt_x = cnt_u; fa.cnt_r = cnt_u; fa.k = k;
        fa.hist_len = H; fa.rre_hist = P->rre.p; fa.res_hist = P->res.p;
        fa.track = track ? 1 : 0; fa.stop_kind = stop_kind; fa.resid_eps = resid_eps; fa.batch = B;
        P->ev_begin(KC_FINALIZE);
        launch_finalize(fa, s);
        P->ev_end();
        P->check_launch();
        if (want_xh) {
          launch_select_copy(P->X3.p, P->st, 0, B, N, P->xh.p + (size_t)(k - 1) * cnt, s);
          ++P->launches;
        }
        if (k < total) cg_direction(0);
        return;
      }
      if (use_precond) {
        P->blur(P->r.p, SEL_EXPLICIT, P->s.p, SEL_EXPLICIT, true, BLUR_STORE, nullptr, nullptr,
                SEL_EXPLICIT, nullptr, 0.0, P->st, pt, KC_BLUR_ADJ);
        cnt_x = P->apply_D(P->s.p, SEL_EXPLICIT, P->X3.p, SEL_NXT, SPEC_AXPY, P->X3.p, SEL_CUR, fd, tau,
                           P->st, pt);
      } else {
        cnt_x = P->blur(P->r.p, SEL_EXPLICIT, P->X3.p, SEL_NXT, true, BLUR_AXPY, nullptr, P->X3.p,
                        SEL_CUR, fd, tau, P->st, pt, KC_BLUR_ADJ);
      }
      const int cnt_r = P->blur(P->X3.p, SEL_NXT, P->r.p, SEL_EXPLICIT, false, BLUR_RESID, gd,
                                nullptr, SEL_EXPLICIT, nullptr, 0.0, P->st, pt, KC_BLUR);
      FinalizeArgs fa{};
      fa.st = P->st; fa.part = pt; fa.cnt_x = cnt_x; fa.cnt_r = cnt_r; fa.k = k;
      fa.hist_len = H; fa.rre_hist = P->rre.p; fa.res_hist = P->res.p;
      fa.track = track ? 1 : 0; fa.stop_kind = stop_kind; fa.resid_eps = resid_eps; fa.batch = B;
      P->ev_begin(KC_FINALIZE);
      launch_finalize(fa, s);
      P->ev_end();
      P->check_launch();
      if (want_xh) {
        launch_select_copy(P->X3.p, P->st, 0, B, N, P->xh.p + (size_t)(k - 1) * cnt, s);
        ++P->launches;
      }
    };

    if (total > 0) {
      // Graph path: one graph per run shape, replayed; kernels read the run's
      // buffers through stable plan-owned pointers.
      char key[640];
      snprintf(key, sizeof key, "%d|%d|%d|%.17g|%.17g|%d|%d|%p|%p|%d|%d|%d|%d|%p|%p|%zu|%llu", total, use_precond,
               stop_kind, resid_eps, tau, (int)track, (int)want_xh, (const void*)gd,
               (const void*)fd, P->conv, P->dst, (int)fused, method, (const void*)P->d, (const void*)P->dT.p,
               P->dstride, (unsigned long long)P->dgen);
      const bool use_graph = !P->timing;
      if (use_graph) {
        if (!P->gexec || P->gkey != key) {
          if (P->gexec) {
            cudaGraphExecDestroy(P->gexec);
            P->gexec = nullptr;
          }
          cudaGraph_t graph;
          const int64_t before = P->launches;
          ck(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal), "capture");
          try {
            enqueue_pre();
            for (int k = 1; k <= total; ++k) enqueue(k);
          } catch (...) {
            // never leave the plan's stream in capture mode
            cudaGraph_t broken = nullptr;
            cudaStreamEndCapture(s, &broken);
            if (broken) cudaGraphDestroy(broken);
            cudaGetLastError();
            throw;
          }
          ck(cudaStreamEndCapture(s, &graph), "end capture");
          ck(cudaGraphInstantiate(&P->gexec, graph, 0), "instantiate");
          cudaGraphDestroy(graph);
          P->glaunches = P->launches - before;  // kernels per replay
          P->launches = before;
          P->gkey = key;
        }
        ck(cudaGraphLaunch(P->gexec, s), "graph launch");
        P->launches += P->glaunches;
      } else {
        enqueue_pre();
        for (int k = 1; k <= total; ++k) enqueue(k);
      }
    }

    // ---- outputs ----
    double* rd = is_device_ptr(restored) ? restored : nullptr;
    if (!rd) {
      P->out.ensure(cnt);
      rd = P->out.p;
    }
    if (total > 0) {
      launch_select_copy(P->X3.p, P->st, (stop_kind == DBX_STOP_MINRRE && track) ? 1 : 0, B, N, rd, s);
      ++P->launches;
    } else {
      ck(cudaMemsetAsync(rd, 0, cnt * sizeof(double), s), "memset");
    }
    P->check_launch();
    stage_out(P, restored, rd, cnt);
    std::vector<ImgState> hs((size_t)B);
    ck(cudaMemcpyAsync(hs.data(), P->st, sizeof(ImgState) * B, cudaMemcpyDeviceToHost, s), "D2H");
    if (total > 0) {
      if (res_hist) stage_out(P, res_hist, P->res.p, (size_t)B * H);
      if (rre_hist && track) stage_out(P, rre_hist, P->rre.p, (size_t)B * H);
    }
    if (want_xh && total > 0) {
      if (is_device_ptr(x_hist)) {
        for (int b = 0; b < B; ++b)
          for (int k = 0; k < total; ++k)
            ck(cudaMemcpyAsync(x_hist + ((size_t)b * H + k) * N, P->xh.p + ((size_t)k * B + b) * N,
                               N * sizeof(double), cudaMemcpyDeviceToDevice, s), "copy");
      } else {
        for (int b = 0; b < B; ++b)
          for (int k = 0; k < total; ++k)
            ck(cudaMemcpyAsync(x_hist + ((size_t)b * H + k) * N, P->xh.p + ((size_t)k * B + b) * N,
                               N * sizeof(double), cudaMemcpyDeviceToHost, s), "D2H");
      }
    }
    ck(cudaStreamSynchronize(s), "sync");
    P->ev_collect();
    int div_img = -1, div_k = 0;
    for (int b = 0; b < B; ++b) {
      // the minimum-RRE buffer only matters under MinRre; a run without any
      // iteration keeps x_0 = 0 (handled above)
      const ImgState& h = hs[(size_t)b];
      if (best_iter) best_iter[b] = total > 0 ? h.best_iter : 0;
      if (iters_done) iters_done[b] = total > 0 ? h.iters : 0;
      if (total > 0 && h.done == 2 && div_img < 0) {
        div_img = b;
        div_k = h.diverged_at;
      }
    }
    // rre() throws on a zero true image (image.hpp:89); the device loop ran
    // with ||f|| = 0, so its histories are meaningless: report the reference's
    // error instead of returning them
    if (track && total > 0)
      for (int b = 0; b < B; ++b) require(hs[(size_t)b].f_norm > 0.0, "rre: zero true image");
    if (div_img >= 0) {
      char msg[160];
      snprintf(msg, sizeof msg, "landweber: iterate exceeded 1e8 * ||g|| (image %d, iteration %d)",
               img_base + div_img, div_k);
      throw Diverged(msg);
    }
  });
}

// Chunked batch run with host<->device copies overlapped with compute: chunk
// c's inputs go up on a copy stream ahead of time, its solve waits only for its
// own inputs, and its restored images come down while chunk c+1 computes.
// Results are those of dbx_landweber_run on the concatenated batch (every
// image is independent; each plan computes its chunk bit-identically).
int dbx_landweber_run_chunks(dbx_plan* const* plans, int nplans, const double* g, const double* f_true,
                             double tau, int max_iters, int stop_kind, int fixed_iters, double resid_eps,
                             int use_precond, double* restored, double* rre_hist, double* res_hist,
                             int* best_iter, int* iters_done) {
  int first_div = DBX_OK;
  std::string div_msg;
  const int st = guarded([&] {
    require(plans && nplans >= 1, "landweber_chunks: no plans");
    require(g && restored, "landweber_chunks: null argument");
    for (int c = 0; c < nplans; ++c) {
      require(plans[c] != nullptr, "landweber_chunks: null plan");
      require(plans[c]->n1 == plans[0]->n1 && plans[c]->n2 == plans[0]->n2 && plans[c]->device == plans[0]->device,
              "landweber_chunks: plans must share the image size and device");
    }
    require(!is_device_ptr(g) && !is_device_ptr(restored) && (!f_true || !is_device_ptr(f_true)),
            "landweber_chunks: g, f_true and restored are host arrays (use dbx_landweber_run for device data)");
    plans[0]->set_dev();
    const int total = stop_kind == DBX_STOP_FIXED ? fixed_iters : max_iters;
    const size_t H = (size_t)std::max(total, 1);
    const size_t N = plans[0]->N;
    cudaStream_t cs = nullptr;
    std::vector<cudaEvent_t> ready((size_t)nplans, nullptr);
    auto cleanup = [&] {
      for (cudaEvent_t e : ready)
        if (e) cudaEventDestroy(e);
      if (cs) cudaStreamDestroy(cs);
    };
    try {
      ck(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking), "stream");
      size_t off = 0;
      for (int c = 0; c < nplans; ++c) {  // every chunk's inputs queued up front, in chunk order
        dbx_plan* P = plans[c];
        const size_t cnt = N * P->batch;
        P->g.ensure(cnt);
        ck(cudaMemcpyAsync(P->g.p, g + off, cnt * sizeof(double), cudaMemcpyHostToDevice, cs), "H2D");
        if (f_true) {
          P->f.ensure(cnt);
          ck(cudaMemcpyAsync(P->f.p, f_true + off, cnt * sizeof(double), cudaMemcpyHostToDevice, cs), "H2D");
        }
        ck(cudaEventCreateWithFlags(&ready[(size_t)c], cudaEventDisableTiming), "event");
        ck(cudaEventRecord(ready[(size_t)c], cs), "event");
        off += cnt;
      }
      // the chunks' solves run concurrently (one host thread per plan: the
      // call is host-synchronous), so one chunk's kernel tails overlap the
      // others' work; each chunk's restored images go down on its own stream
      std::vector<size_t> first((size_t)nplans + 1, 0);
      for (int c = 0; c < nplans; ++c) {
        plans[c]->out.ensure(N * plans[c]->batch);
        first[(size_t)c + 1] = first[(size_t)c] + (size_t)plans[c]->batch;
      }
      std::vector<int> rcs((size_t)nplans, DBX_OK);
      std::vector<std::string> msgs((size_t)nplans);
      // at most `depth` chunks solve at once (chunk c starts when chunk
      // c - depth has finished): concurrent chunks share the GPU and would all
      // finish together, leaving every download for the end; a bounded
      // pipeline finishes them in order, so all but the last downloads
      // overlap the remaining solves
      static const int depth = [] {
        const char* e = std::getenv("DBX_CHUNK_DEPTH");
        const int v = e ? std::atoi(e) : 2;
        return v < 1 ? 1 : v;
      }();
      std::vector<std::promise<void>> fin((size_t)nplans);
      std::vector<std::shared_future<void>> fin_f;
      for (auto& pr : fin) fin_f.push_back(pr.get_future().share());
      auto work = [&](int c) {
        if (c >= depth) fin_f[(size_t)(c - depth)].wait();
        dbx_plan* P = plans[c];
        const size_t img = first[(size_t)c], cnt = N * P->batch;
        int rc = DBX_OK;
        if (cudaSetDevice(P->device) != cudaSuccess || cudaStreamWaitEvent(P->stream, ready[(size_t)c], 0) != cudaSuccess) {
          rc = DBX_ECUDA;
          g_err = "landweber_chunks: stream setup failed";
        } else {
          rc = run_impl(P, P->g.p, f_true ? P->f.p : nullptr, tau, max_iters, stop_kind, fixed_iters, resid_eps,
                        use_precond, P->out.p, rre_hist ? rre_hist + img * H : nullptr,
                        res_hist ? res_hist + img * H : nullptr, best_iter ? best_iter + img : nullptr,
                        iters_done ? iters_done + img : nullptr, nullptr, 0, (int)img);
        }
        if (rc == DBX_OK || rc == DBX_EDIVERGED) {  // restored images exist either way
          if (cudaMemcpyAsync(restored + img * N, P->out.p, cnt * sizeof(double), cudaMemcpyDeviceToHost,
                              P->stream) != cudaSuccess ||
              cudaStreamSynchronize(P->stream) != cudaSuccess) {
            rc = DBX_ECUDA;
            g_err = "landweber_chunks: D2H failed";
          }
        }
        rcs[(size_t)c] = rc;
        msgs[(size_t)c] = g_err;  // g_err is per thread
        fin[(size_t)c].set_value();
      };
      std::vector<std::thread> pool;
      for (int c = 1; c < nplans; ++c) pool.emplace_back(work, c);
      work(0);
      for (std::thread& t : pool) t.join();
      for (int c = 0; c < nplans; ++c) {
        const int rc = rcs[(size_t)c];
        if (rc == DBX_EINVAL) throw InvalidArg(msgs[(size_t)c]);
        if (rc != DBX_OK && rc != DBX_EDIVERGED) throw CudaErr(msgs[(size_t)c]);
      }
      for (int c = 0; c < nplans && first_div == DBX_OK; ++c)
        if (rcs[(size_t)c] == DBX_EDIVERGED) {
          first_div = DBX_EDIVERGED;
          div_msg = msgs[(size_t)c];
        }
      ck(cudaStreamSynchronize(cs), "sync");
    } catch (...) {
      if (cs) cudaStreamSynchronize(cs);
      cleanup();
      throw;
    }
    cleanup();
  });
  if (st != DBX_OK) return st;
  if (first_div != DBX_OK) {
    g_err = div_msg;
    return first_div;
  }
  return DBX_OK;
}


// ---------------------------------------------------------------------------
// NCCL communicators and the C++ row-slab loop (see the section header above
// `struct dbx_slab`).
// ---------------------------------------------------------------------------
int dbx_comm_unique_id(unsigned char* id) {
  return guarded([&] {
    require(id != nullptr, "comm_unique_id: null argument");
    NcclApi& n = nccl_api();
    if (!n.ok) throw CudaErr(n.why);
    ncclUniqueId u;
    nck(n.GetUniqueId(&u), "ncclGetUniqueId");
    static_assert(sizeof(u.internal) == DBX_COMM_ID_BYTES, "ncclUniqueId size");
    std::memcpy(id, u.internal, DBX_COMM_ID_BYTES);
  });
}

int dbx_comm_init(int nranks, const unsigned char* id, int rank, int device, dbx_comm** out) {
  return guarded([&] {
    require(out && id && nranks >= 1 && rank >= 0 && rank < nranks, "comm_init: bad argument");
    *out = nullptr;
    NcclApi& n = nccl_api();
    if (!n.ok) throw CudaErr(n.why);
    ck(cudaSetDevice(device), "cudaSetDevice");
    ncclUniqueId u;
    std::memcpy(u.internal, id, DBX_COMM_ID_BYTES);
    auto c = std::make_unique<dbx_comm>();
    nck(n.CommInitRank(&c->comm, nranks, u, rank), "ncclCommInitRank");
    c->nranks = nranks;
    c->rank = rank;
    c->owned = true;
    *out = c.release();
  });
}

int dbx_comm_wrap(void* nccl_comm, int nranks, int rank, dbx_comm** out) {
  return guarded([&] {
    require(out && nccl_comm && nranks >= 1 && rank >= 0 && rank < nranks, "comm_wrap: bad argument");
    auto c = std::make_unique<dbx_comm>();
    c->comm = static_cast<ncclComm_t>(nccl_comm);
    c->nranks = nranks;
    c->rank = rank;
    *out = c.release();
  });
}

void dbx_comm_destroy(dbx_comm* c) {
  if (!c) return;
  if (c->owned && c->comm && nccl_api().ok) nccl_api().CommDestroy(c->comm);
  delete c;
}

int dbx_slab_create(int n, int parts, int rank, const double* taps, int q1, int q2, double alpha, dbx_comm* comm,
                    int device, dbx_slab** out) {
  return guarded([&] {
    require(out != nullptr, "slab_create: null out");
    *out = nullptr;
    require(n >= 3 && parts >= 1 && n % parts == 0, "row slabs: image rows must divide evenly across ranks");
    require(alpha >= 0.0, "tikhonov_filter: alpha must be nonnegative");
    require(rank < parts, "slab_create: rank out of range");
    if (rank >= 0 && parts > 1) {
      require(comm != nullptr, "slab_create: a rank of a multi-rank decomposition needs a communicator");
      require(comm->nranks == parts && comm->rank == rank, "slab_create: communicator does not match (parts, rank)");
    }
    const int R = n / parts;
    require(R >= q1 + 1, "row slabs: every slab needs at least q + 1 rows (the global AR extension is local)");
    auto S = std::make_unique<dbx_slab>();
    S->n = n; S->P = parts; S->q = q1; S->R = R; S->C = R; S->device = device;
    S->nloc = rank < 0 ? parts : 1;
    S->rank0 = rank < 0 ? 0 : rank;
    S->comm = (rank >= 0 && parts > 1) ? comm : nullptr;
    dbx_plan* h = nullptr;
    const int rc = dbx_plan_create(R, n, 1, taps, q1, q2, DBX_BC_ANTIREFLECTIVE, device, &h);
    if (rc != DBX_OK) {
      if (rc == DBX_EINVAL) throw InvalidArg(g_err);
      throw CudaErr(g_err);
    }
    S->plan = h;
    dbx_plan* P = h;
    P->set_dev();
    if (P->conv == DBX_CONV_DIRECT || !P->use_fft_conv()) P->conv = DBX_CONV_FFT;
    require(P->use_fft_conv(), "slab_create: no compiled FFT correlation length for this slab");
    P->ensure_conv();
    S->sep = P->sep_direct(BLUR_RESID);
    P->blue_tables(1, false);  // throws when no DST core exists for the row length
    const size_t slab = (size_t)R * n, nl = (size_t)S->nloc;
    for (DevBuf* b : {&S->x, &S->best, &S->r, &S->s, &S->u, &S->tA, &S->tB}) b->ensure(nl * slab);
    if (parts > 1)
      for (DevBuf* b : {&S->send, &S->recv}) b->ensure(nl * slab);
    S->top.ensure(nl * q1 * n);
    S->bot.ensure(nl * q1 * n);
    if (!S->sep) S->ext.ensure((size_t)(R + 2 * q1) * n);
    P->zb.ensure(std::max((size_t)(R + 2 * q1) * n, (size_t)(R + 2 * q1) * P->Lh * 2));
    S->part.ensure(nl * NUM_SLOTS * (size_t)P->part_cap);
    S->tot.ensure(nl * 4);
    ck(cudaMalloc(&S->st, sizeof(ImgState)), "cudaMalloc");
    // this process's blocks of d^T: rows c in [p C, (p+1) C) of d^T (columns of d)
    S->dTb.ensure(nl * slab);
    int* flag = nullptr;
    ck(cudaMalloc(&flag, sizeof(int)), "cudaMalloc");
    ck(cudaMemsetAsync(flag, 0, sizeof(int), P->stream), "memset");
    for (int i = 0; i < S->nloc; ++i)
      launch_build_filter_block(P->sym, q1, q2, n, n, alpha, 0, n, (S->rank0 + i) * S->C, S->C, 1,
                                S->dTb.p + (size_t)i * slab, flag, P->stream, 0);
    int hflag = 0;
    ck(cudaMemcpyAsync(&hflag, flag, sizeof(int), cudaMemcpyDeviceToHost, P->stream), "D2H");
    ck(cudaStreamSynchronize(P->stream), "sync");
    cudaFree(flag);
    require(alpha > 0.0 || hflag == 0, "tikhonov_filter: alpha = 0 with a zero eigenvalue");
    *out = S.release();
  });
}

void dbx_slab_destroy(dbx_slab* S) { delete S; }

int dbx_slab_set_iterates(dbx_slab* S, double* buf, int count) {
  return guarded([&] {
    require(S != nullptr && count >= 0, "slab_set_iterates: bad argument");
    require(!buf || is_device_ptr(buf), "slab_set_iterates: device pointer");
    S->keep = count > 0 ? buf : nullptr;
    S->keep_n = buf ? count : 0;
  });
}

void* dbx_slab_stream(dbx_slab* S) { return S ? (void*)S->plan->stream : nullptr; }

int dbx_slab_info(dbx_slab* S, int* rows, int* local_slabs, int* separable, int64_t* launches) {
  return guarded([&] {
    require(S != nullptr, "slab_info: null slab");
    if (rows) *rows = S->R;
    if (local_slabs) *local_slabs = S->nloc;
    if (separable) *separable = S->sep ? 1 : 0;
    if (launches) *launches = S->plan->launches;
  });
}

int dbx_slab_run(dbx_slab* S, const double* g, const double* f, double tau, int max_iters, int stop_kind,
                 double resid_eps, double* x_out, double* rre_hist, double* res_hist, int* best_iter,
                 int* iters_done) {
  return guarded([&] {
    require(S && g && x_out && best_iter && iters_done, "slab_run: null argument");
    require(max_iters >= 1, "SolverConfig: max_iters must be >= 1");
    require(stop_kind >= DBX_STOP_FIXED && stop_kind <= DBX_STOP_RESIDUAL, "slab_run: unknown stopping rule");
    require(stop_kind != DBX_STOP_MINRRE || f, "StoppingRule::MinRre needs the true image");
    require(is_device_ptr(g) && is_device_ptr(x_out) && (!f || is_device_ptr(f)), "slab_run: device pointers");
    dbx_plan* P = S->plan;
    P->set_dev();
    const cudaStream_t st = P->stream;
    const int n = S->n, R = S->R, C = S->C, q = S->q, PP = S->P, nl = S->nloc;
    const size_t slab = (size_t)R * n, cap = (size_t)P->part_cap;
    const bool track = f != nullptr;
    NcclApi* nc = S->comm ? &nccl_api() : nullptr;
    if (S->comm && !nc->ok) throw CudaErr(nc->why);
    auto part_of = [&](int i) { return Partials{S->part.p + (size_t)i * NUM_SLOTS * cap, (int)cap}; };
    auto tot_of = [&](int i) { return S->tot.p + (size_t)i * 4; };
    auto allreduce = [&] {
      if (nc) nck(nc->AllReduce(S->tot.p, S->tot.p, 3, ncclDouble, ncclSum, S->comm->comm, st), "ncclAllReduce");
      else if (nl > 1) launch_slab_local_allreduce(S->tot.p, nl, 4, st);
    };
    int64_t& L = P->launches;
    // ---- exchanges ----------------------------------------------------------
    // halo views for slab i of buffer b: the neighbours' edge rows (in-process:
    // their memory; NCCL: received into top/bot) or the global AR rows
    std::vector<const double*> htop(nl), hbot(nl);
    auto halos = [&](double* b) {
      for (int i = 0; i < nl; ++i) {
        const int p = S->rank0 + i;
        double* bi = b + (size_t)i * slab;
        double* ti = S->top.p + (size_t)i * q * n;
        double* oi = S->bot.p + (size_t)i * q * n;
        if (nc) {
          nck(nc->GroupStart(), "ncclGroupStart");
          if (p > 0) {
            nck(nc->Send(bi, (size_t)q * n, ncclDouble, p - 1, S->comm->comm, st), "ncclSend");
            nck(nc->Recv(ti, (size_t)q * n, ncclDouble, p - 1, S->comm->comm, st), "ncclRecv");
          }
          if (p + 1 < PP) {
            nck(nc->Send(bi + (size_t)(R - q) * n, (size_t)q * n, ncclDouble, p + 1, S->comm->comm, st), "ncclSend");
            nck(nc->Recv(oi, (size_t)q * n, ncclDouble, p + 1, S->comm->comm, st), "ncclRecv");
          }
          nck(nc->GroupEnd(), "ncclGroupEnd");
          htop[i] = ti;
          hbot[i] = oi;
        } else {
          htop[i] = p > 0 ? bi - (size_t)q * n : ti;
          hbot[i] = p + 1 < PP ? bi + slab : oi;
        }
        if (p == 0 || p + 1 == PP) {
          launch_slab_ar_halo(bi, R, n, q, p == 0 ? ti : nullptr, p + 1 == PP ? oi : nullptr, st);
          ++L;
        }
      }
    };
    // all-to-all of nl x P chunks of R x C doubles (send -> recv)
    auto all2all = [&] {
      const size_t chunk = (size_t)R * C;
      if (nc) {
        nck(nc->GroupStart(), "ncclGroupStart");
        for (int s = 0; s < PP; ++s) {
          nck(nc->Send(S->send.p + s * chunk, chunk, ncclDouble, s, S->comm->comm, st), "ncclSend");
          nck(nc->Recv(S->recv.p + s * chunk, chunk, ncclDouble, s, S->comm->comm, st), "ncclRecv");
        }
        nck(nc->GroupEnd(), "ncclGroupEnd");
      } else {
        for (int p = 0; p < nl; ++p)
          for (int s = 0; s < PP; ++s)
            ck(cudaMemcpyAsync(S->recv.p + (size_t)s * slab + p * chunk, S->send.p + (size_t)p * slab + s * chunk,
                               chunk * sizeof(double), cudaMemcpyDeviceToDevice, st), "all-to-all copy");
      }
    };
    auto pack = [&](const double* src, double* blocks, bool unpack) {  // slab (R x n) <-> P blocks of R x C
      const size_t w = (size_t)C * sizeof(double), pitch = (size_t)n * sizeof(double);
      for (int s = 0; s < PP; ++s) {
        double* blk = blocks + (size_t)s * R * C;
        double* col = const_cast<double*>(src) + (size_t)s * C;
        if (unpack) ck(cudaMemcpy2DAsync(col, pitch, blk, w, w, R, cudaMemcpyDeviceToDevice, st), "unpack");
        else ck(cudaMemcpy2DAsync(blk, w, col, pitch, w, R, cudaMemcpyDeviceToDevice, st), "pack");
      }
    };
    // ---- blur of every local slab: y = A b (adjoint = 0, residual with g) or A' b
    auto blur = [&](double* b, double* y, bool adjoint, bool resid) {
      halos(b);
      int cnt = 0;
      for (int i = 0; i < nl; ++i) {
        SpecArgs a = P->spec_base(S->st, part_of(i));
        P->set_kernel(a.conv, adjoint);
        a.conv.tw1 = reinterpret_cast<const double2*>(P->tw1);
        a.conv.tw2 = reinterpret_cast<const double2*>(P->tw2);
        a.conv.L1 = P->L1; a.conv.L2 = P->L2; a.conv.Lh = P->Lh;
        a.zbuf = reinterpret_cast<double2*>(P->zb.p);
        a.ybuf = reinterpret_cast<double2*>(P->yb.p);
        a.out = y + (size_t)i * slab;
        a.g = resid ? g + (size_t)i * slab : nullptr;
        if (S->sep) {
          a.in = b + (size_t)i * slab;
          a.halo = q; a.htop = htop[i]; a.hbot = hbot[i];
          lc(launch_rows_sep_seg(a, st), "rows_sep_seg");
          cnt = lc(launch_cols_sep_epi(a, resid ? 1 : 0, st), "cols_sep_real");
          L += 2;
        } else {
          double* e = S->ext.p;
          ck(cudaMemcpyAsync(e, htop[i], (size_t)q * n * sizeof(double), cudaMemcpyDeviceToDevice, st), "ext");
          ck(cudaMemcpyAsync(e + (size_t)q * n, b + (size_t)i * slab, slab * sizeof(double), cudaMemcpyDeviceToDevice,
                             st), "ext");
          ck(cudaMemcpyAsync(e + (size_t)(q + R) * n, hbot[i], (size_t)q * n * sizeof(double),
                             cudaMemcpyDeviceToDevice, st), "ext");
          a.in = e;
          a.n1 = R + 2 * q;
          lc(launch_conv_row_fwd(a, st), "launch_conv_row_fwd");
          a.n1 = R;
          a.preext = 1;
          lc(launch_conv_col(a, st), "launch_conv_col");
          a.preext = 0;
          a.epi = resid ? SPEC_RESID : SPEC_STORE;
          cnt = lc(launch_conv_row_inv(a, st), "launch_conv_row_inv");
          L += 3;
        }
      }
      P->check_launch();
      return cnt;
    };
    auto rows = [&](int kind, const double* in, double* out, int rows_n, int i, int epi, const double* aux,
                    const double* ff, int kind2) {
      SpecArgs a = P->spec_base(S->st, part_of(i));
      a.blue2 = P->blue_tables(1, false);
      a.n1 = rows_n;
      a.in = in; a.out = out; a.kind1 = kind; a.kind2 = kind2;
      a.epi = epi;
      a.d = epi == SPEC_HADAMARD || kind2 >= 0 ? aux : nullptr;
      a.dstride = 0;
      a.xold = epi == SPEC_AXPY ? aux : nullptr;
      a.f = ff;
      a.tau = tau;
      ++L;
      return lc(launch_dst_rows(a, st), "launch_dst_rows");
    };
    // ---- ||g||, ||f||, state -------------------------------------------------
    for (int i = 0; i < nl; ++i) {
      const int k = launch_slab_sumsq(g + (size_t)i * slab, f ? f + (size_t)i * slab : nullptr, slab, part_of(i), st);
      launch_slab_tot(part_of(i), k, 0, 1, tot_of(i), nullptr, st);
      L += 2;
    }
    allreduce();
    launch_slab_state_init(S->st, S->tot.p, st);
    ++L;
    if (track) {  // rre() throws on a zero true image (image.hpp:89)
      ImgState h;
      ck(cudaMemcpyAsync(&h, S->st, sizeof h, cudaMemcpyDeviceToHost, st), "D2H");
      ck(cudaStreamSynchronize(st), "sync");
      require(h.f_norm > 0.0, "rre: zero true image");
    }
    S->hist.ensure(2 * (size_t)max_iters);
    ck(cudaMemsetAsync(S->x.p, 0, nl * slab * sizeof(double), st), "memset");
    ck(cudaMemcpyAsync(S->r.p, g, nl * slab * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy");
    for (int k = 1; k <= max_iters; ++k) {
      // s = A' r, then T~ along the rows into u
      blur(S->r.p, S->s.p, true, false);
      for (int i = 0; i < nl; ++i)
        rows(DBX_KIND_ARINV, S->s.p + i * slab, S->u.p + i * slab, R, i, SPEC_STORE, nullptr, nullptr, -1);
      // column half of D on the transposed column blocks: T~, x d^T, T in one pass
      if (PP == 1) {
        launch_transpose(S->u.p, S->tA.p, R, n, st);
        rows(DBX_KIND_ARINV, S->tA.p, S->tB.p, C, 0, SPEC_STORE, S->dTb.p, nullptr, DBX_KIND_AR);
        launch_transpose(S->tB.p, S->s.p, C, n, st);
        L += 2;
      } else {
        for (int i = 0; i < nl; ++i) pack(S->u.p + i * slab, S->send.p + i * slab, false);
        all2all();
        for (int i = 0; i < nl; ++i) {  // recv: n x C (rows stacked by source slab) -> C x n
          launch_transpose(S->recv.p + i * slab, S->tA.p + i * slab, n, C, st);
          rows(DBX_KIND_ARINV, S->tA.p + i * slab, S->tB.p + i * slab, C, i, SPEC_STORE, S->dTb.p + i * slab, nullptr,
               DBX_KIND_AR);
          launch_transpose(S->tB.p + i * slab, S->send.p + i * slab, C, n, st);
          L += 2;
        }
        all2all();
        for (int i = 0; i < nl; ++i) pack(S->s.p + i * slab, S->recv.p + i * slab, true);
      }
      // T along the rows, x_k = x_{k-1} + tau (.) in place, ||x||^2 and ||x - f||^2 partials
      int cnt_x = 0;
      for (int i = 0; i < nl; ++i)
        cnt_x = rows(DBX_KIND_AR, S->s.p + i * slab, S->x.p + i * slab, R, i, SPEC_AXPY, S->x.p + i * slab,
                     f ? f + i * slab : nullptr, -1);
      // r = g - A x_k with ||r||^2 partials
      const int cnt_r = blur(S->x.p, S->r.p, false, true);
      for (int i = 0; i < nl; ++i) launch_slab_tot(part_of(i), cnt_x, cnt_r, track ? 1 : 0, tot_of(i), S->st, st);
      allreduce();
      launch_slab_finalize(S->st, S->tot.p, k, track ? S->hist.p : nullptr, S->hist.p + max_iters, track ? 1 : 0,
                           stop_kind, resid_eps, st);
      L += nl + 1;
      if (track) {
        launch_slab_best_copy(S->st, S->x.p, S->best.p, nl * slab, st);
        ++L;
      }
      if (S->keep && k <= S->keep_n)
        ck(cudaMemcpyAsync(S->keep + (size_t)(k - 1) * nl * slab, S->x.p, nl * slab * sizeof(double),
                           cudaMemcpyDeviceToDevice, st), "keep iterate");
      P->check_launch();
    }
    ImgState h;
    ck(cudaMemcpyAsync(&h, S->st, sizeof h, cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    const int done = h.done == 2 ? h.diverged_at - 1 : h.iters;
    const double* src = (track && h.best_iter > 0) ? S->best.p : S->x.p;
    ck(cudaMemcpyAsync(x_out, src, nl * slab * sizeof(double), cudaMemcpyDeviceToDevice, st), "copy");
    std::vector<double> hh(2 * (size_t)max_iters);
    ck(cudaMemcpyAsync(hh.data(), S->hist.p, hh.size() * sizeof(double), cudaMemcpyDeviceToHost, st), "D2H");
    ck(cudaStreamSynchronize(st), "sync");
    if (rre_hist && track) std::memcpy(rre_hist, hh.data(), sizeof(double) * (size_t)std::max(done, 0));
    if (res_hist) std::memcpy(res_hist, hh.data() + max_iters, sizeof(double) * (size_t)std::max(done, 0));
    *best_iter = h.best_iter;
    *iters_done = done;
    if (h.done == 2) {
      char msg[160];
      snprintf(msg, sizeof msg, "landweber: iterate exceeded 1e8 * ||g|| (row slabs, iteration %d)", h.diverged_at);
      throw Diverged(msg);
    }
  });
}

}  // extern "C"
