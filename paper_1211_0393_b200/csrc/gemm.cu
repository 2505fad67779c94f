// gemm.cu — K3/K4 dense form: the 1D AR transforms T~_n / T_n (and the plain
// DST-I Q_n) applied to every column (C = M X) or every row (C = X M^T) of a
// batch of images as an FP64 GEMM on the tensor cores, with fused epilogues.
//
// Replaces (reference): sine1_forward + r2r_run(RODFT00) transforms.hpp:114-121,
// ar_forward / ar_inverse transforms.hpp:148-173, tensor_map transforms.hpp:179-192,
// the Hadamard by d in filter_apply spectral.hpp:163, and x += tau*step plus
// the iterate norms of solver.hpp:104-117.
//
// The dense matrices carry the rank-2 border corrections in their first/last
// columns (dense_ar_forward / dense_ar_inverse block forms), so one GEMM pass
// is exactly one reference tensor_map half-pass.
//
// Engine: FP64 DMMA (`mma.sync.aligned.m8n8k4.row.col.f64`).  sm_100a has no
// FP64 kind in tcgen05 (ptxas rejects .kind::f64), so the warp-level DMMA is
// the FP64 tensor path on B200: one instruction = 256 FMAs (8x the DFMA work
// per issue slot).  A CTA of 128 threads (2 x 2 warps) computes a BM x BN
// tile; every warp holds (BM/2) x (BN/2) as (BM/16) x (BN/16) 8x8 accumulators.
// K advances in slabs of 16 through a 3-deep cp.async ring:
//   As[BM][16+4]  row-major (A fragment A[gid][tig]: conflict-free, stride 20),
//   Bs[16][BN+4]  row-major (B fragment B[tig][gid]: conflict-free, stride BN+4).
// Fragment layouts (PTX ISA, mma.m8n8k4 .f64): A row = gid, col = tig;
// B row = tig, col = gid; C rows gid, cols 2 tig + {0,1}; gid = lane/4,
// tig = lane%4.  Accumulation order inside one output: k ascending in steps
// of 4, each DMMA sums its 4 products in hardware order — not the FFTW order,
// which parity (1e-10 per iterate) does not depend on.
#include <cuda_runtime.h>

#include "dbx_internal.h"

namespace dbx {

namespace {

constexpr int kThreads = 128;
constexpr int BK = 16;
constexpr int kStages = 3;

__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, bool valid) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const int sz = valid ? 8 : 0;  // src-size 0 zero-fills the slot
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(sz));
}
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ double block_sum(double v, double* red) {
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

template <int BM, int BN>
struct Smem {
  double A[kStages][BM][BK + 4];
  double B[kStages][BK][BN + 4];
  double red[kThreads / 32];
};

template <int BM, int BN>
__global__ void __launch_bounds__(kThreads) gemm_dmma_kernel(GemmArgs a) {
  DBX_PDL_WAIT();
  constexpr int WM = BM / 2, WN = BN / 2;     // warp tile
  constexpr int TMI = WM / 8, TNI = WN / 8;   // 8x8 accumulators per warp
  const int b = blockIdx.z;
  if (a.st && a.st[b].done) return;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  Smem<BM, BN>& sm = *reinterpret_cast<Smem<BM, BN>*>(smem_raw);

  const double* A = (a.asel == SEL_EXPLICIT) ? a.A + (long long)b * a.sA
                                             : resolve_ptr(a.A, a.st, a.asel, b, a.batch, a.img_elems);
  const double* B = (a.bsel == SEL_EXPLICIT) ? a.B + (long long)b * a.sB
                                             : resolve_ptr(a.B, a.st, a.bsel, b, a.batch, a.img_elems);
  const int M = a.M, N = a.N, K = a.K;
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gid = lane >> 2, tig = lane & 3;
  const int wm0 = (warp >> 1) * WM, wn0 = (warp & 1) * WN;
  // 16-byte copies when every row of both operands starts 16-byte aligned
  const bool vec = ((K | N) & 1) == 0 && ((reinterpret_cast<size_t>(A) | reinterpret_cast<size_t>(B)) & 15) == 0;

  auto load_stage = [&](int st, int k0) {
    if (vec && k0 + BK <= K) {
      // A: BM rows x 16 doubles = BM*8 16-byte chunks
#pragma unroll
      for (int e = threadIdx.x; e < BM * (BK / 2); e += kThreads) {
        const int mm = e / (BK / 2), kk = (e % (BK / 2)) * 2;
        const int gm = m0 + mm;
        if (gm < M) cp_async16(&sm.A[st][mm][kk], A + (long long)gm * K + k0 + kk);
        else { sm.A[st][mm][kk] = 0.0; sm.A[st][mm][kk + 1] = 0.0; }
      }
    } else {
#pragma unroll
      for (int e = threadIdx.x; e < BM * BK; e += kThreads) {
        const int mm = e / BK, kk = e % BK;
        const int gm = m0 + mm, gk = k0 + kk;
        const bool ok = gm < M && gk < K;
        cp_async8(&sm.A[st][mm][kk], ok ? A + (long long)gm * K + gk : A, ok);
      }
    }
    if (vec && n0 + BN <= N) {
#pragma unroll
      for (int e = threadIdx.x; e < BK * (BN / 2); e += kThreads) {
        const int kk = e / (BN / 2), nn = (e % (BN / 2)) * 2;
        const int gk = k0 + kk;
        if (gk < K) cp_async16(&sm.B[st][kk][nn], B + (long long)gk * N + n0 + nn);
        else { sm.B[st][kk][nn] = 0.0; sm.B[st][kk][nn + 1] = 0.0; }
      }
    } else {
#pragma unroll
      for (int e = threadIdx.x; e < BK * BN; e += kThreads) {
        const int kk = e / BN, nn = e % BN;
        const int gk = k0 + kk, gn = n0 + nn;
        const bool ok = gk < K && gn < N;
        cp_async8(&sm.B[st][kk][nn], ok ? B + (long long)gk * N + gn : B, ok);
      }
    }
  };

  double acc[TMI][TNI][2];
#pragma unroll
  for (int i = 0; i < TMI; ++i)
#pragma unroll
    for (int j = 0; j < TNI; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nk = (K + BK - 1) / BK;
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nk) load_stage(s, s * BK);
    cp_commit();
  }
  for (int kt = 0; kt < nk; ++kt) {
    cp_wait<kStages - 2>();
    __syncthreads();
    // refill the stage consumed two steps ago (every warp is past it)
    const int nxt = kt + kStages - 1;
    if (nxt < nk) load_stage(nxt % kStages, nxt * BK);
    cp_commit();
    const int st = kt % kStages;
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[TMI], bf[TNI];
#pragma unroll
      for (int i = 0; i < TMI; ++i) af[i] = sm.A[st][wm0 + 8 * i + gid][ks + tig];
#pragma unroll
      for (int j = 0; j < TNI; ++j) bf[j] = sm.B[st][ks + tig][wn0 + 8 * j + gid];
#pragma unroll
      for (int i = 0; i < TMI; ++i)
#pragma unroll
        for (int j = 0; j < TNI; ++j) dmma(acc[i][j], af[i], bf[j]);
    }
  }
  cp_wait<0>();

  // ---- epilogue ----
  double* C = (a.csel == SEL_EXPLICIT)
                  ? a.C + (long long)b * a.sC
                  : const_cast<double*>(resolve_ptr(a.C, a.st, a.csel, b, a.batch, a.img_elems));
  const double* xo = a.epi == EPI_AXPY ? resolve_ptr(a.xold, a.st, a.xoldsel, b, a.batch, a.img_elems) : nullptr;
  const double* f = (a.epi == EPI_AXPY && a.f) ? a.f + (size_t)b * a.img_elems : nullptr;
  const double* d = a.epi == EPI_HADAMARD ? a.d + (size_t)b * a.dstride : nullptr;
  double p0 = 0.0, p1 = 0.0;
#pragma unroll
  for (int i = 0; i < TMI; ++i) {
    const int gm = m0 + wm0 + 8 * i + gid;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < TNI; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn0 + 8 * j + 2 * tig + h;
        if (gn >= N) continue;
        const long long o = (long long)gm * N + gn;
        double v = acc[i][j][h];
        if (a.epi == EPI_HADAMARD) {
          v *= d[o];
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
  }
  if (a.epi == EPI_AXPY && a.part.p) {
    const int cta = blockIdx.y * gridDim.x + blockIdx.x;
    double* P = a.part.p + (size_t)b * NUM_SLOTS * a.part.cap;
    const double s0 = block_sum(p0, sm.red);
    if (threadIdx.x == 0) P[SLOT_X2 * a.part.cap + cta] = s0;
    const double s1 = block_sum(p1, sm.red);
    if (threadIdx.x == 0) P[SLOT_XF2 * a.part.cap + cta] = s1;
  }
}

template <int BM, int BN>
void launch_tile(const GemmArgs& a, cudaStream_t s, int* ctas_per_image) {
  const size_t smem = sizeof(Smem<BM, BN>);
  static AttrOnce once;
  once.ensure(gemm_dmma_kernel<BM, BN>, smem);
  dim3 grid((a.N + BN - 1) / BN, (a.M + BM - 1) / BM, a.batch);
  if (ctas_per_image) *ctas_per_image = grid.x * grid.y;
  launch_k(gemm_dmma_kernel<BM, BN>, grid, kThreads, smem, s, a);
}

}  // namespace

void launch_gemm(const GemmArgs& a, cudaStream_t s, int* ctas_per_image) {
  // Large tiles while they still fill two waves of 148 SMs; small tiles for
  // small single images (C1: 256^2 -> 64 CTAs of 32 x 32).
  const long long t64 = (long long)((a.M + 63) / 64) * ((a.N + 63) / 64) * a.batch;
  const long long t32x64 = (long long)((a.M + 31) / 32) * ((a.N + 63) / 64) * a.batch;
  if (t64 >= 2 * 148)
    launch_tile<64, 64>(a, s, ctas_per_image);
  else if (t32x64 >= 148)
    launch_tile<32, 64>(a, s, ctas_per_image);
  else
    launch_tile<32, 32>(a, s, ctas_per_image);
}

}  // namespace dbx
