// spectral.h — argument blocks and launchers of the FFT-form kernels
// (spectral.cu): FFT-correlation blur and Bluestein DST-I / AR transforms.
#pragma once

#include <cuda_runtime.h>

#include "../../include/dbx.h"
#include "dbx_internal.h"
#include "radix.h"

namespace dbx {

// Column convolutions of the FFT-form blur (conv_col) run the in-place
// Cooley-Tukey core with the kernel spectrum in digit-reversed order (the host
// permutes each column, dbx_api.cu ensure_conv); -DDBX_CONV_STOCKHAM keeps
// forward + inverse Stockham FFTs with the spectrum in natural order (A/B).
#ifdef DBX_CONV_STOCKHAM
constexpr bool kConvCt = false;
#else
constexpr bool kConvCt = true;
#endif


// N-point DFT core of the packed DST (dst.cu): direct (M = N smooth),
// Bluestein (M = 2^k >= 2N-1), Rader (M = N-1, N prime).
// CORE_PFA: prime factor N = N1 N2 (Good-Thomas), row DFTs of N1 in
// registers, column DFTs of the prime N2 by Rader (C4: 2047 = 23 x 89).
enum DstCore { CORE_DIRECT = 0, CORE_BLUE = 1, CORE_RADER = 2, CORE_PFA = 3 };

enum SpecEpi { SPEC_STORE = 0, SPEC_HADAMARD = 1, SPEC_RESID = 2, SPEC_AXPY = 3 };

// FFT-correlation tables (device): twiddles W_L^e for L1/L2 and the kernel
// spectrum H[k2][k1] = conj(FFT2(w))[k1][k2] / (L1 L2), k2 < Lh = L2/2 + 1.
struct ConvTables {
  const double2* tw1 = nullptr;
  const double2* tw2 = nullptr;
  const double2* H = nullptr;
  int L1 = 0, L2 = 0, Lh = 0;
  // rank-1 mask w = a b^T (conv_col_sep): column taps a (2 q1 + 1) and the
  // row factor's spectrum beta(k2) = conj(B(k2)) / L2 (Lh); null = full H
  const double* sepa = nullptr;
  const double2* sepb = nullptr;
  const double* sepr = nullptr;  // row taps b (2 q2 + 1): direct row pass of the separable fused pipeline
  const double* sepa_host = nullptr;  // host copy of sepa: cols_sep_real takes its taps as kernel parameters
  // row taps b by value (q2 <= 15): part of the kernel parameter block, so the
  // direct row passes' DFMAs read them from the constant bank, not registers
  double sepr_v[31] = {};
};

// Bluestein DST-I tables for one line length n (device): M-point twiddles,
// chirp w_j = exp(-i pi j^2 / N) (j < N), kernel spectrum FFT_M(conj chirp)/M,
// the AR ramp p_j = 1 - j/(n-1) and alpha_n (transforms.hpp:135-144).
struct BlueTables {
  const double2* tw = nullptr;
  const double2* chirp = nullptr;
  const double2* bhat = nullptr;
  const double2* bct = nullptr;  // bhat at the in-place Cooley-Tukey core's digit-reversed positions
  const double2* bctT = nullptr; // bct element-major [r][block] (unpadded 8190-point CT line: coalesced product pass)
  const double2* tw1t = nullptr; // warp-owned DFT_1023 / DFT_255: level-1 twiddles [k1][32 lanes] (tables.h)
  const double* p = nullptr;
  const double* sn = nullptr;  // sin(pi j / N), j < N (packed real DST)
  const int* dlog = nullptr;   // Rader: position of z_j (discrete log base g), j in [1, N)
  const int* ridx = nullptr;   // Rader: position of Z_l in the convolution output, l in [1, N)
  int core = 0;                // DstCore
  double rinv = 1.0;  // 1 / (n - 1): ramp p_j = 1 - j rinv computed in registers
  double c0 = 0.0;    // DCT (CosineIII): sqrt(1/m) for k = 0 (scale = sqrt(2/m) otherwise)
  double alpha = 1.0;
  double scale = 1.0;  // sqrt(2/N)
  int n = 0, N = 0, M = 0;
};

struct SpecArgs {
  const double* in = nullptr; int insel = SEL_EXPLICIT;
  double* out = nullptr; int outsel = SEL_EXPLICIT;
  int n1 = 0, n2 = 0, q1 = 0, q2 = 0, batch = 0;
  int epi = SPEC_STORE;
  int bc = DBX_BC_ANTIREFLECTIVE;                // blur extension (boundary.hpp:33-64)
  const double* g = nullptr;                     // RESID
  const double* xold = nullptr; int xoldsel = SEL_EXPLICIT;  // AXPY
  const double* f = nullptr;                     // AXPY (nullable)
  const double* d = nullptr;                     // HADAMARD / dst_cols middle
  double tau = 0.0;
  const ImgState* st = nullptr;
  Partials part{nullptr, 0};
  // FFT correlation
  ConvTables conv;
  double2* zbuf = nullptr;                       // [batch][n1][Lh], or [batch][Lh][n1] if ztrans
  double2* ybuf = nullptr;                       // [batch][n1][Lh]
  int ztrans = 0;                                // fused pipeline: row-FFT spectra stored transposed
  int preext = 0;                                // conv_col: n1 + 2 q1 input rows already extended (row slabs)
  // row slabs, separable direct blur: halo = q1 rows above (htop) and below
  // (hbot) the slab's n1 rows; rows_sep_seg then correlates n1 + 2 halo rows
  // into Z^T (column stride n1 + 2 halo) and cols_sep_real reads them as the
  // vertical extension instead of synthesising it
  int halo = 0;
  const double* htop = nullptr;
  const double* hbot = nullptr;
  const double* dT = nullptr;                    // d transposed [n2][n1] (fused column pass)
  size_t dstride = 0;                            // filter grid per image (alpha sweep) or shared (0)
  // DST
  int kind1 = DBX_KIND_ARINV, kind2 = -1;
  int pf = 0;                                    // dst_rows: prefetch the rows of CTA blockIdx.x + pf into L2 (0: off)
  int tout = 0;                                  // dst_rows, SPEC_STORE: write the output transposed, out[k * n1 + row]
  // residual kernels of the fused pipelines: when fin_cnt is set, the last
  // CTA of each image runs the iteration's finalize (finalize.cuh) — one
  // launch fewer per iteration
  FinalizeArgs fin{};
  unsigned* fin_cnt = nullptr;
  BlueTables blue1;                              // columns (length n1)
  BlueTables blue2;                              // rows (length n2)
};

// Row stride (complex elements) of the column-pass output Y: Lh rounded up to
// even so a row pair of adjacent columns is one 32-byte aligned store.
__host__ __device__ constexpr int y_stride(int Lh) { return (Lh + 1) & ~1; }

int conv_supported_len(int need);   // smallest compiled L >= need, 0 if none
int blue_supported_len(int need);   // smallest compiled power of two M >= need, 0 if none
int conv_rows_per_cta(int L2);
int direct_supported_len(int N);  // N if the direct odd-length DFT is compiled, else 0
int rader_supported_len(int M);   // M (= N-1) if the Rader convolution length is compiled, else 0
int pfa_supported_len(int N);     // N if the prime-factor core is compiled for N, else 0 (pfa_factors gives N1, N2)
void pfa_factors(int N, int* N1, int* N2);

// Each returns the number of CTAs per image (for the partial-sum count), -1 if
// the size is not compiled.
int launch_conv_row_fwd(const SpecArgs& a, cudaStream_t s);
int launch_conv_col(const SpecArgs& a, cudaStream_t s);  // conv_col, or conv_col_sep when conv.sepa is set
bool conv_sep_supported(int q1);                         // conv_col_sep compiled for this q1
int launch_conv_row_inv(const SpecArgs& a, cudaStream_t s);
int launch_dst_rows(const SpecArgs& a, cudaStream_t s);
// CosineIII transforms along rows (dct.cu): kind1 = +1 forward R (DCT-II),
// -1 inverse R^T (DCT-III); blue2 carries the DCT tables (chirp = e^{-i pi k / 2m}).
int launch_dct_rows(const SpecArgs& a, cudaStream_t s);
int dct_supported_len(int m);
int launch_dst_cols(const SpecArgs& a, cudaStream_t s);

// Fused row pipelines of the preconditioned iteration (fused.cu).
// *_SEP: the separable (rank-1 mask) pipeline's row kernels — direct row
// passes instead of the row FFTs (Z'^T / Y real, row-major Y).
enum FusedKind {
  FUSED_AINV_TT = 0, FUSED_T_AXPY_AFWD = 1, FUSED_AINV_RESID = 2, FUSED_DST_TCOLS = 3,
  FUSED_TT_SEP = 4, FUSED_T_AXPY_SEP = 5, FUSED_RESID_SEP = 6
};
bool fused_supported(int L2, int M, bool bluestein);
bool fused_sep_supported(int L2, int M, bool bluestein, int n2, int q2);
int launch_cols_sep_real(const SpecArgs& a, cudaStream_t s);  // real column pass of the separable pipeline
// separate-pass direct separable blur: row pass (any n2) -> Z^T, then the
// column pass with a store (resid = 0) or residual r = g - Y (resid = 1) epilogue
bool rows_sep_supported(int q2);
int launch_rows_sep_seg(const SpecArgs& a, cudaStream_t s);
int launch_cols_sep_epi(const SpecArgs& a, int resid, cudaStream_t s);
int launch_fused(int which, const SpecArgs& a, cudaStream_t s);
// wdst.cu: warp-owned column half of D for 1024-point columns (-1: not this shape)
int launch_dst_tcols_w(const SpecArgs& a, cudaStream_t s);
// wdst.cu: warp-owned separable-pipeline row kernels for 1024-point rows
// (which 0: rows_tt_w = K2, 1: rows_t_axpy_w = K4; -1: not this shape)
int launch_rows_w(int which, const SpecArgs& a, cudaStream_t s);
#ifdef DBX_PHASES
int fused_debug_phases(unsigned long long* out, int n);  // read + reset (instrumented builds)
#endif

}  // namespace dbx
