// finalize.cuh — the per-iteration loop bookkeeping of the reference
// (landweber_loop, solver.hpp:101-131) as a device function: fixed-order
// reduction of the fused-epilogue norm partials, divergence guard, histories,
// strict-'<' best-RRE tracking on the iterate ring, residual rule.  Used by
// finalize_kernel (solver_kernels.cu) and, as a last-block tail, by the
// residual kernels of the fused pipelines (fused.cu), which saves one launch
// per iteration.
#pragma once

#include <cuda_runtime.h>
#include <math.h>

#include "dbx_internal.h"

namespace dbx {

// The three fixed-order block sums of finalize in one pass: the same per-thread
// strided order and the same shuffle tree as partial_sum / block_reduce (the
// results are bit-identical), with all three slots' loads in flight together
// and one barrier pair instead of three.
__device__ __forceinline__ void block_reduce3(double& a, double& b, double& c) {
  __shared__ double red3[3][32];
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_xor_sync(0xffffffffu, a, o);
    b += __shfl_xor_sync(0xffffffffu, b, o);
    c += __shfl_xor_sync(0xffffffffu, c, o);
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) {
    red3[0][w] = a;
    red3[1][w] = b;
    red3[2][w] = c;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double sa = 0.0, sb = 0.0, sc = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) {
      sa += red3[0][i];
      sb += red3[1][i];
      sc += red3[2][i];
    }
    a = sa;
    b = sb;
    c = sc;
  }
}

// Reduce the fused-epilogue partials of iteration k for image b and apply
// the reference loop bookkeeping (solver.hpp:107-124), with every thread of
// the calling CTA.  cnt_r < 0: the residual partials come from the calling
// kernel itself (last-block finalize, finalize_last_block) — its gridDim.x.
// Partials are read through L2 (__ldcg): other CTAs of the same launch may
// have written them.
__device__ __forceinline__ void finalize_image(const FinalizeArgs& a, int b) {
  ImgState* st = a.st + b;
  const ImgState s0 = *st;  // in flight with the partial loads
  if (s0.done) return;
  const double* P = a.part.p + (size_t)b * NUM_SLOTS * a.part.cap;
  const int cnt_r = a.cnt_r < 0 ? (int)gridDim.x : a.cnt_r;
  double x2 = 0.0, xf2 = 0.0, r2 = 0.0;
  for (int i = threadIdx.x; i < a.cnt_x; i += blockDim.x) x2 += __ldcg(P + SLOT_X2 * a.part.cap + i);
  if (a.track)
    for (int i = threadIdx.x; i < a.cnt_x; i += blockDim.x) xf2 += __ldcg(P + SLOT_XF2 * a.part.cap + i);
  for (int i = threadIdx.x; i < cnt_r; i += blockDim.x) r2 += __ldcg(P + SLOT_R2 * a.part.cap + i);
  block_reduce3(x2, xf2, r2);
  if (threadIdx.x != 0) return;
  ImgState s = s0;
  const int k = a.k;
  const double xn = sqrt(x2);
  // divergence guard before recording (solver.hpp:107-108)
  if (xn > 1e8 * s.g_norm && s.g_norm > 0.0) {
    s.done = 2;
    s.diverged_at = k;
    s.cur = s.nxt;
    *st = s;
    return;
  }
  const double rn = sqrt(r2);
  if (a.res_hist) a.res_hist[(size_t)b * a.hist_len + (k - 1)] = rn;
  if (a.track) {
    const double e = sqrt(xf2) / s.f_norm;
    if (a.rre_hist) a.rre_hist[(size_t)b * a.hist_len + (k - 1)] = e;
    if (e < s.best_rre) {  // strict '<': first minimum wins (solver.hpp:114)
      s.best_rre = e;
      s.best_iter = k;
      s.best = s.nxt;
    }
  }
  s.iters = k;
  // rotate buffers: x_k becomes current; next target avoids cur and best
  s.cur = s.nxt;
  int n = 0;
  while (n == s.cur || n == s.best) ++n;
  s.nxt = n;
  if (a.stop_kind == 2 && s.g_norm > 0.0 && rn / s.g_norm < a.resid_eps) s.done = 1;
  *st = s;
}


// Last-block finalize: every CTA of image b (blockIdx.y) has written its
// residual partial (thread 0) when it calls this; the CTA that arrives last
// runs finalize_image for the image and re-arms the counter.  All threads of
// every CTA must call it (no early return after the kernel's done check).
__device__ __forceinline__ void finalize_last_block(const FinalizeArgs& a, unsigned* counter, int b) {
  __shared__ int is_last;
  __threadfence();  // this CTA's partial write is visible before it is counted
  __syncthreads();
  if (threadIdx.x == 0) is_last = atomicAdd(counter + b, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!is_last) return;
  __threadfence();
  finalize_image(a, b);
  if (threadIdx.x == 0) counter[b] = 0;
}

}  // namespace dbx
