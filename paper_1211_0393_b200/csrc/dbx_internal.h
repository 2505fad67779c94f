// dbx_internal.h — device-side data structures and kernel launchers of the
// B200 AR-deblurring path (see DESIGN.md for the data layout in HBM).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <string>
#include <vector>

namespace dbx {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: one bit per
// device ordinal, set on the first launch on that device.  Thread-safe
// (racing first launches both set the attribute, which is idempotent), so
// plans on several GPUs in one process, and the chunk worker threads of
// dbx_landweber_run_chunks, all see the attribute on their own device.
struct AttrOnce {
  std::atomic<unsigned long long> done{0};
  template <typename K>
  bool ensure(K kernel, size_t bytes) {
    if (bytes > 227 * 1024) return false;
    if (bytes <= 48 * 1024) return true;
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    const unsigned long long bit = 1ull << (dev & 63);
    if (done.load(std::memory_order_acquire) & bit) return true;
    if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes) != cudaSuccess)
      return false;
    done.fetch_or(bit, std::memory_order_acq_rel);
    return true;
  }
};

// ---- programmatic dependent launch (PDL) ------------------------------------
// Every kernel of the solver loop starts with DBX_PDL_WAIT(): wait until the
// previous grid of the stream has completed and its memory is visible, then
// let the next grid begin launching.  Launched through launch_k (attribute
// cudaLaunchAttributeProgrammaticStreamSerialization; captured into the CUDA
// graph as programmatic edges), a kernel's CTAs are scheduled onto the SMs
// the previous kernel's tail leaves idle and sit at the wait, so the launch
// latency and prologue of every node overlap the previous node's drain —
// the per-node gap that dominates small images (C1: 7 nodes per iteration).
// A plainly launched kernel passes the wait immediately.
#define DBX_PDL_WAIT()                                      \
  do {                                                      \
    asm volatile("griddepcontrol.wait;" ::: "memory");      \
    asm volatile("griddepcontrol.launch_dependents;" ::);   \
  } while (0)

bool pdl_enabled();  // DBX_PDL=1 turns the attribute on (off by default: measured slower)

template <typename... KP, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KP...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                            Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// Per-image iteration state, resident in HBM for the whole run.  The three
// iterate buffers X[0..2] are used round-robin so that tracking the best
// iterate (solver.hpp:111-119) never copies x: `best` pins a buffer, `cur`
// holds x_{k-1}, `nxt` receives x_k.
struct ImgState {
  int cur, best, nxt;
  int done;         // 0 running, 1 residual rule hit, 2 diverged
  int iters;        // iterations executed (solver.hpp:120)
  int best_iter;    // 1-based, 0 = none
  int diverged_at;  // first iteration whose ||x|| > guard
  int pad_;
  double best_rre;
  double g_norm, f_norm;
};

enum BufSel { SEL_EXPLICIT = -1, SEL_CUR = 0, SEL_NXT = 2 };

// Partial-sum slots written by the fused epilogues and reduced (fixed order,
// deterministic) by the finalize kernel.
enum Slot { SLOT_X2 = 0, SLOT_XF2 = 1, SLOT_R2 = 2, NUM_SLOTS = 3 };

struct Partials {
  double* p;      // [batch][NUM_SLOTS][cap]
  int cap;        // entries per (image, slot)
};

__host__ __device__ inline const double* resolve_ptr(const double* base, const ImgState* st,
                                                     int sel, int b, int batch, size_t N) {
#ifdef __CUDA_ARCH__
  if (sel == SEL_EXPLICIT) return base + (size_t)b * N;
  const int idx = sel == SEL_CUR ? st[b].cur : st[b].nxt;
  return base + ((size_t)idx * batch + b) * N;
#else
  (void)st; (void)sel;
  return base + (size_t)b * N;
#endif
}

// ---- blur (AR stencil) --------------------------------------------------
enum BlurMode { BLUR_STORE = 0, BLUR_RESID = 1, BLUR_AXPY = 2 };

struct BlurArgs {
  const double* x; int xsel;          // input image(s)
  double* y; int ysel;                // output (STORE/RESID: explicit; AXPY: x_nxt)
  const double* w;                    // correlation weights (2q1+1)(2q2+1), oriented
  int n1, n2, q1, q2, batch;
  int mode;
  int bc;                             // DBX_BC_ANTIREFLECTIVE / DBX_BC_REFLECTIVE
  const double* g;                    // RESID: data
  const double* xold; int xoldsel;    // AXPY: x_{k-1}
  const double* f;                    // AXPY: true image (nullable)
  double tau;
  const ImgState* st;                 // nullable outside the solver
  Partials part;
};
void launch_blur(const BlurArgs& a, cudaStream_t s, int* ctas_per_image);

// ---- dense-form AR transform passes (FP64 GEMM with fused epilogues) ----
enum GemmEpi { EPI_STORE = 0, EPI_HADAMARD = 1, EPI_AXPY = 2 };

struct GemmArgs {
  // C[b] (M x N) = A[b] (M x K) * B[b] (K x N), row-major.
  const double* A; long long sA; int asel;
  const double* B; long long sB; int bsel;
  double* C; long long sC; int csel;
  int M, N, K, batch;
  int epi;
  const double* d;                    // HADAMARD: M x N filter grid (shared, or per image: dstride)
  size_t dstride;
  const double* xold; int xoldsel;    // AXPY
  const double* f;                    // AXPY (nullable)
  double tau;
  const ImgState* st;
  Partials part;
  size_t img_elems;                   // n1*n2 (for buffer resolution)
};
void launch_gemm(const GemmArgs& a, cudaStream_t s, int* ctas_per_image);

// ---- GPU-side input synthesis (gen_dev.cu) --------------------------------
// Status DBX_* with the message in err (the C-ABI wrappers set dbx_last_error).
int mt19937_64_device(uint64_t seed, uint64_t count, uint64_t* out, int device, std::string& err);
int gen_honest_device(int rows, int cols, int nshapes, double sinus_amp, uint64_t scene_seed, const double* taps,
                      int q1, int q2, int n1, int n2, double noise_level, uint64_t noise_seed, double* f_true,
                      double* g, int device, std::string& err);

// ---- spectrum, norms, finalize -----------------------------------------
// grid 0: anti-reflective grid, 1: reflective (DCT-III) grid
void launch_build_filter(const double* sym_taps, int q1, int q2, int n1, int n2, double alpha,
                         double* d, int* zero_flag, cudaStream_t s, int grid = 0);
void launch_build_filter_block(const double* sym_taps, int q1, int q2, int n1, int n2, double alpha, int r0,
                               int nr, int c0, int nc, int tr, double* d, int* zero_flag, cudaStream_t s,
                               int grid = 0);
void launch_norms_init(const double* g, const double* f, int batch, size_t N, ImgState* st, Partials pt,
                       cudaStream_t s);
struct FinalizeArgs {
  ImgState* st;
  Partials part;
  int cnt_x, cnt_r;       // partial counts per image for the x- and r-norm slots
  int k;                  // 1-based iteration index
  int hist_len;
  double* rre_hist;       // [batch][hist_len] (device)
  double* res_hist;
  int track, stop_kind;
  double resid_eps;
  int batch;
};
void launch_finalize(const FinalizeArgs& a, cudaStream_t s);
void launch_state_init(ImgState* st, int batch, cudaStream_t s);
void launch_select_copy(const double* X3, const ImgState* st, int which_best, int batch,
                        size_t N, double* out, cudaStream_t s);
void launch_zero(double* p, size_t n, cudaStream_t s);

// ---- reblurred (preconditioned) CGLS scalars and vector steps (cg.cu) ----
struct CgScalars {
  double gamma, alpha, beta, pad_;
};
void launch_cg_alpha(const ImgState* st, CgScalars* cs, Partials pt, int cnt, int batch, cudaStream_t s);
int launch_cg_update(const double* X3, const ImgState* st, const CgScalars* cs, const double* p, const double* qn,
                     double* r, const double* f, int batch, size_t N, Partials pt, cudaStream_t s);
int launch_cg_dot(const ImgState* st, const double* a, const double* b, int batch, size_t N, double* part, int cap,
                  cudaStream_t s);
void launch_cg_beta(const ImgState* st, CgScalars* cs, const double* part, int cap, int cnt, int init, int batch,
                    cudaStream_t s);
void launch_cg_xpay(const ImgState* st, const CgScalars* cs, const double* z, double* p, int batch, size_t N,
                    cudaStream_t s);
void launch_slab_ar_rows(const double* x, double* ext, int rows, int n2, int q, int top, int bot, cudaStream_t s);
void launch_transpose(const double* in, double* out, int rows, int cols, cudaStream_t s, int batch = 1);
// C++ row-slab loop (dbx_slab_run)
void launch_slab_ar_halo(const double* x, int rows, int n2, int q, double* top, double* bot, cudaStream_t s);
int launch_slab_sumsq(const double* g, const double* f, size_t n, Partials pt, cudaStream_t s);
void launch_slab_tot(Partials pt, int cnt_x, int cnt_r, int track, double* tot, const ImgState* st, cudaStream_t s);
void launch_slab_local_allreduce(double* tots, int parts, int stride, cudaStream_t s);
void launch_slab_state_init(ImgState* st, const double* tot2, cudaStream_t s);
void launch_slab_finalize(ImgState* st, const double* tot, int k, double* rre_hist, double* res_hist, int track,
                          int stop_kind, double eps, cudaStream_t s);
void launch_slab_best_copy(const ImgState* st, const double* x, double* best, size_t n, cudaStream_t s);

}  // namespace dbx
