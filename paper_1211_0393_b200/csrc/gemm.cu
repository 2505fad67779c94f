// gemm.cu — K3/K4 dense form: the 1D AR transforms T~_n / T_n (and the plain
// DST-I Q_n) applied to every column (C = M X) or every row (C = X M^T) of a
// batch of images as an FP64 GEMM with fused epilogues.
//
// Replaces (reference): sine1_forward + r2r_run(RODFT00) transforms.hpp:114-121,
// ar_forward / ar_inverse transforms.hpp:148-173, tensor_map transforms.hpp:179-192,
// the Hadamard by d in filter_apply spectral.hpp:163, and x += tau*step plus
// the iterate norms of solver.hpp:104-117.
//
// The dense matrices carry the rank-2 border corrections in their first/last
// columns (dense_ar_forward / dense_ar_inverse block forms), so one GEMM pass
// is exactly one reference tensor_map half-pass.  Register-blocked SIMT FP64:
// a CTA of 256 threads computes a BM x BN tile, each thread TM x TN outputs on
// a 16 x 16 thread grid with stride-16 interleave (conflict-free smem reads).
#include <cuda_runtime.h>

#include "dbx_internal.h"

namespace dbx {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double block_sum256(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0)
    for (int i = 0; i < kThreads / 32; ++i) s += red[i];
  return s;
}

template <int TM, int TN, int BK>
__global__ void __launch_bounds__(kThreads) gemm_kernel(GemmArgs a) {
  constexpr int BM = 16 * TM, BN = 16 * TN;
  const int b = blockIdx.z;
  if (a.st && a.st[b].done) return;
  __shared__ double As[2][BK][BM];
  __shared__ double Bs[2][BK][BN];
  __shared__ double red[kThreads / 32];

  const double* A = (a.asel == SEL_EXPLICIT) ? a.A + (long long)b * a.sA
                                             : resolve_ptr(a.A, a.st, a.asel, b, a.batch, a.img_elems);
  const double* B = (a.bsel == SEL_EXPLICIT) ? a.B + (long long)b * a.sB
                                             : resolve_ptr(a.B, a.st, a.bsel, b, a.batch, a.img_elems);
  const int M = a.M, N = a.N, K = a.K;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;

  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;

  constexpr int A_PER = BM * BK / kThreads;
  constexpr int B_PER = BN * BK / kThreads;
  double ra[A_PER], rb[B_PER];

  auto load_regs = [&](int k0) {
#pragma unroll
    for (int t = 0; t < A_PER; ++t) {
      const int e = threadIdx.x + t * kThreads;
      const int mm = e / BK, kk = e - mm * BK;
      const int gm = m0 + mm, gk = k0 + kk;
      ra[t] = (gm < M && gk < K) ? A[(long long)gm * K + gk] : 0.0;
    }
#pragma unroll
    for (int t = 0; t < B_PER; ++t) {
      const int e = threadIdx.x + t * kThreads;
      const int kk = e / BN, nn = e - kk * BN;
      const int gk = k0 + kk, gn = n0 + nn;
      rb[t] = (gk < K && gn < N) ? B[(long long)gk * N + gn] : 0.0;
    }
  };
  auto store_smem = [&](int buf) {
#pragma unroll
    for (int t = 0; t < A_PER; ++t) {
      const int e = threadIdx.x + t * kThreads;
      const int mm = e / BK, kk = e - mm * BK;
      As[buf][kk][mm] = ra[t];
    }
#pragma unroll
    for (int t = 0; t < B_PER; ++t) {
      const int e = threadIdx.x + t * kThreads;
      const int kk = e / BN, nn = e - kk * BN;
      Bs[buf][kk][nn] = rb[t];
    }
  };

  const int nk = (K + BK - 1) / BK;
  load_regs(0);
  store_smem(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) load_regs((kt + 1) * BK);
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      double av[TM], bv[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) av[i] = As[buf][kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < TN; ++j) bv[j] = Bs[buf][kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) acc[i][j] = fma(av[i], bv[j], acc[i][j]);
    }
    if (kt + 1 < nk) store_smem(buf ^ 1);
    __syncthreads();
  }

  // ---- epilogue ----
  double* C = (a.csel == SEL_EXPLICIT)
                  ? a.C + (long long)b * a.sC
                  : const_cast<double*>(resolve_ptr(a.C, a.st, a.csel, b, a.batch, a.img_elems));
  const double* xo = a.epi == EPI_AXPY ? resolve_ptr(a.xold, a.st, a.xoldsel, b, a.batch, a.img_elems) : nullptr;
  const double* f = (a.epi == EPI_AXPY && a.f) ? a.f + (size_t)b * a.img_elems : nullptr;
  double p0 = 0.0, p1 = 0.0;
#pragma unroll
  for (int i = 0; i < TM; ++i) {
    const int gm = m0 + ty + 16 * i;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TN; ++j) {
      const int gn = n0 + tx + 16 * j;
      if (gn >= N) continue;
      const long long o = (long long)gm * N + gn;
      double v = acc[i][j];
      if (a.epi == EPI_HADAMARD) {
        v *= a.d[(size_t)b * a.dstride + o];
      } else if (a.epi == EPI_AXPY) {
        v = xo[o] + a.tau * v;
        p0 += v * v;
        if (f) {
          const double e = v - f[o];
          p1 += e * e;
        }
      }
      C[o] = v;
    }
  }
  if (a.epi == EPI_AXPY && a.part.p) {
    const int cta = blockIdx.y * gridDim.x + blockIdx.x;
    double* P = a.part.p + (size_t)b * NUM_SLOTS * a.part.cap;
    const double s0 = block_sum256(p0, red);
    if (threadIdx.x == 0) P[SLOT_X2 * a.part.cap + cta] = s0;
    const double s1 = block_sum256(p1, red);
    if (threadIdx.x == 0) P[SLOT_XF2 * a.part.cap + cta] = s1;
  }
}

}  // namespace

void launch_gemm(const GemmArgs& a, cudaStream_t s, int* ctas_per_image) {
  // Large tiles for large operands; small tiles keep >= 1 wave on 148 SMs for
  // small single images.
  const long long tiles128 = (long long)((a.M + 127) / 128) * ((a.N + 127) / 128) * a.batch;
  if (tiles128 >= 148) {
    dim3 grid((a.N + 127) / 128, (a.M + 127) / 128, a.batch);
    if (ctas_per_image) *ctas_per_image = grid.x * grid.y;
    gemm_kernel<8, 8, 8><<<grid, kThreads, 0, s>>>(a);
  } else {
    dim3 grid((a.N + 63) / 64, (a.M + 63) / 64, a.batch);
    if (ctas_per_image) *ctas_per_image = grid.x * grid.y;
    gemm_kernel<4, 4, 16><<<grid, kThreads, 0, s>>>(a);
  }
}

}  // namespace dbx
