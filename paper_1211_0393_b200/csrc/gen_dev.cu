// gen_dev.cu — GPU-side Honest synthesis: the seeded scene,
// the Honest blur-then-crop and add_noise for the large canvases (C5: 8222^2)
// that take seconds on the host.
//
// Restated reference pieces: synthesize Honest branch (experiment.hpp:71-99:
// centred offsets, margin >= q, direct correlation g(r,c) = sum_s h_s
// scene(off + (r,c) - s), crop), add_noise + GaussianSampler (image.hpp:44-82:
// std::mt19937_64(seed), u1 = ((r>>11)+1) 2^-53, u2 = (r>>11) 2^-53, the pair
// r cos(2 pi u2), r sin(2 pi u2), eta rescaled to level * ||g|| / ||eta||).
//
// Kernels:
//   paint      one thread per canvas pixel; the shapes overlapping its 32x32
//              tile (host-built CSR lists, generation order) are scanned from
//              the last one back, the first covering shape gives the value
//              (painter's rule).  The in/out test uses the host painter's exact
//              IEEE operations (__dmul_rn/__dadd_rn/__ddiv_rn: no contraction;
//              gen.cpp is compiled with -ffp-contract=off), so the scene — and
//              f_true — equal the host generator's bit for bit.
//   honest     the direct (2q1+1)x(2q2+1) correlation over a staged canvas
//              window, one accumulator in the reference's s1-then-s2 order with
//              separate multiply and add (the host's operations): bit-identical
//              clean image.
//   mt19937_64 one CTA twists the 312-word state per block in two half-steps
//              (words 0..155 read only the old state; words 156..311 also read
//              the new words i-156 and 0) and tempers the block: exactly
//              std::mt19937_64's stream (checked against the host one).
//   noise      Box-Muller per sample pair (device log/sin/cos: within 1 ulp of
//              the host libm), fixed-order two-level norm reductions, g = clean
//              + s eta.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <string>
#include <vector>

#include "../../include/dbx.h"
#include "dbx_internal.h"

namespace dbx {

namespace {

constexpr int kTile = 32;
constexpr double kPi = 3.141592653589793238462643383279502884;

__global__ void __launch_bounds__(256) paint_kernel(double* __restrict__ out, int rows, int cols,
                                                    const double* __restrict__ prm,
                                                    const int* __restrict__ tstart,
                                                    const int* __restrict__ tlist, int tiles_x, double amp) {
  const int c = blockIdx.x * kTile + threadIdx.x;
  const int tile = blockIdx.y * tiles_x + blockIdx.x;
  const int lo = tstart[tile], hi = tstart[tile + 1];
#pragma unroll 1
  for (int rr = threadIdx.y; rr < kTile; rr += blockDim.y) {
    const int r = blockIdx.y * kTile + rr;
    if (r >= rows || c >= cols) continue;
    double v = 0.0;
    for (int i = hi - 1; i >= lo; --i) {
      const double* P = prm + (size_t)tlist[i] * DBX_SHAPE_PARAMS;
      if (r < (int)P[8] || r > (int)P[9] || c < (int)P[10] || c > (int)P[11]) continue;
      const double cy = P[1], cx = P[2], a = P[3], b = P[4], ct = P[5], st = P[6];
      const double dy = __dadd_rn(__dadd_rn((double)r, 0.5), -cy);
      const double dx = __dadd_rn(__dadd_rn((double)c, 0.5), -cx);
      const double u = __dadd_rn(__dmul_rn(dx, ct), __dmul_rn(dy, st));
      const double w = __dadd_rn(__dmul_rn(-dx, st), __dmul_rn(dy, ct));
      const bool in = P[0] != 0.0
                          ? __dadd_rn(__ddiv_rn(__dmul_rn(u, u), __dmul_rn(a, a)),
                                      __ddiv_rn(__dmul_rn(w, w), __dmul_rn(b, b))) <= 1.0
                          : fabs(u) <= a && fabs(w) <= b;
      if (in) {
        v = P[7];
        break;
      }
    }
    if (amp != 0.0) {
      // amp * sin(2 pi (3 (r + 1/2) / rows + 2 (c + 1/2) / cols)), host order
      const double t1 = __ddiv_rn(__dmul_rn(3.0, __dadd_rn((double)r, 0.5)), (double)rows);
      const double t2 = __ddiv_rn(__dmul_rn(2.0, __dadd_rn((double)c, 0.5)), (double)cols);
      v = __dadd_rn(v, __dmul_rn(amp, sin(__dmul_rn(2.0 * kPi, __dadd_rn(t1, t2)))));
    }
    out[(size_t)r * cols + c] = v;
  }
}

// One output tile TH x 32 per CTA (256 threads: 32 columns x 8 row groups),
// canvas window (TH + 2 q1) x (32 + 2 q2) staged in shared memory.
constexpr int kHTH = 32;
__global__ void __launch_bounds__(256) honest_kernel(const double* __restrict__ scene, int cols,
                                                     const double* __restrict__ taps, int q1, int q2, int n1,
                                                     int n2, int off1, int off2, double* __restrict__ clean,
                                                     double* __restrict__ f_true) {
  extern __shared__ double win[];
  const int W = 2 * q2 + 1;
  const int WR = kHTH + 2 * q1, WC = 32 + 2 * q2;
  double* tp = win + (size_t)WR * WC;
  const int r0 = blockIdx.y * kHTH, c0 = blockIdx.x * 32;
  const int tid = threadIdx.y * 32 + threadIdx.x;
  for (int e = tid; e < (2 * q1 + 1) * W; e += 256) tp[e] = taps[e];
  // window row i <-> canvas row off1 + r0 - q1 + i, col j <-> off2 + c0 - q2 + j
  for (int e = tid; e < WR * WC; e += 256) {
    const int i = e / WC, j = e - i * WC;
    const int rr = r0 - q1 + i, cc = c0 - q2 + j;
    win[e] = (rr < n1 + q1 && cc < n2 + q2) ? scene[(size_t)(off1 + rr) * cols + (off2 + cc)] : 0.0;
  }
  __syncthreads();
  const int c = c0 + threadIdx.x;
  for (int rr = threadIdx.y; rr < kHTH; rr += 8) {
    const int r = r0 + rr;
    if (r >= n1 || c >= n2) continue;
    double acc = 0.0;
    for (int s1 = -q1; s1 <= q1; ++s1) {
      const double* srow = win + (size_t)(rr + q1 - s1) * WC + (threadIdx.x + q2);
      const double* trow = tp + (size_t)(q1 + s1) * W + q2;
      for (int s2 = -q2; s2 <= q2; ++s2) acc = __dadd_rn(acc, __dmul_rn(trow[s2], srow[-s2]));
    }
    clean[(size_t)r * n2 + c] = acc;
    if (f_true) f_true[(size_t)r * n2 + c] = win[(size_t)(rr + q1) * WC + threadIdx.x + q2];
  }
}

__device__ __forceinline__ uint64_t mt_twist(uint64_t cur, uint64_t nxt) {
  const uint64_t x = (cur & 0xFFFFFFFF80000000ull) | (nxt & 0x7FFFFFFFull);
  return (x >> 1) ^ ((x & 1ull) ? 0xB5026F5AA96619E9ull : 0ull);
}
__device__ __forceinline__ uint64_t mt_temper(uint64_t y) {
  y ^= (y >> 29) & 0x5555555555555555ull;
  y ^= (y << 17) & 0x71D67FFFEDA60000ull;
  y ^= (y << 37) & 0xFFF7EEE000000000ull;
  return y ^ (y >> 43);
}

__global__ void __launch_bounds__(312) mt19937_64_kernel(uint64_t seed, uint64_t count, uint64_t* __restrict__ out) {
  __shared__ uint64_t st[2][312];
  const int t = threadIdx.x;
  if (t == 0) {
    st[0][0] = seed;
    for (int i = 1; i < 312; ++i) st[0][i] = 6364136223846793005ull * (st[0][i - 1] ^ (st[0][i - 1] >> 62)) + i;
  }
  __syncthreads();
  int cur = 0;
  for (uint64_t base = 0; base < count; base += 312) {
    const int nx = cur ^ 1;
    if (t < 156) st[nx][t] = st[cur][t + 156] ^ mt_twist(st[cur][t], st[cur][t + 1]);
    __syncthreads();
    if (t >= 156) st[nx][t] = st[nx][t - 156] ^ mt_twist(st[cur][t], t == 311 ? st[nx][0] : st[cur][t + 1]);
    __syncthreads();
    if (base + t < count) out[base + t] = mt_temper(st[nx][t]);
    cur = nx;
  }
}

// eta[2p], eta[2p+1] from words 2p, 2p+1 (GaussianSampler, image.hpp:44-66)
__global__ void box_muller_kernel(const uint64_t* __restrict__ w, size_t n, double* __restrict__ eta) {
  const size_t p = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * p >= n) return;
  const double u1 = __dmul_rn(__dadd_rn((double)(w[2 * p] >> 11), 1.0), 0x1p-53);
  const double u2 = __dmul_rn((double)(w[2 * p + 1] >> 11), 0x1p-53);
  const double r = sqrt(__dmul_rn(-2.0, log(u1)));
  const double a = __dmul_rn(2.0 * kPi, u2);
  eta[2 * p] = __dmul_rn(r, cos(a));
  if (2 * p + 1 < n) eta[2 * p + 1] = __dmul_rn(r, sin(a));
}

constexpr int kRedBlocks = 1184;  // 8 per SM; fixed, so the reduction order is fixed
__global__ void __launch_bounds__(256) sumsq_partial(const double* __restrict__ x, size_t n,
                                                     double* __restrict__ part) {
  __shared__ double red[8];
  double s = 0.0;
  for (size_t i = (size_t)blockIdx.x * 256 + threadIdx.x; i < n; i += (size_t)gridDim.x * 256)
    s = fma(x[i], x[i], s);
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < 8; ++i) t += red[i];
    part[blockIdx.x] = t;
  }
}
__global__ void sum_final(const double* __restrict__ part, int m, double* __restrict__ out) {
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int i = 0; i < m; ++i) t += part[i];
    *out = t;
  }
}

__global__ void add_scaled(const double* __restrict__ clean, const double* __restrict__ eta, size_t n, double s,
                           double* __restrict__ g) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) g[i] = __dadd_rn(clean[i], __dmul_rn(s, eta[i]));
}

struct Dev {
  std::vector<void*> bufs;
  std::string* err;
  bool ok = true;
  void* alloc(size_t bytes) {
    void* p = nullptr;
    if (cudaMalloc(&p, bytes ? bytes : 1) != cudaSuccess) {
      cudaGetLastError();
      ok = false;
      *err = "cudaMalloc failed (" + std::to_string(bytes) + " bytes)";
      return nullptr;
    }
    bufs.push_back(p);
    return p;
  }
  ~Dev() {
    for (void* p : bufs) cudaFree(p);
  }
};

bool on_device(const void* p) {
  cudaPointerAttributes at;
  if (!p || cudaPointerGetAttributes(&at, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return at.type == cudaMemoryTypeDevice || at.type == cudaMemoryTypeManaged;
}

int cuda_status(std::string& err, const char* where) {
  const cudaError_t e = cudaGetLastError();
  if (e == cudaSuccess) return DBX_OK;
  err = std::string(where) + ": " + cudaGetErrorString(e);
  return DBX_ECUDA;
}

int mt_stream(uint64_t seed, uint64_t count, uint64_t* dst, cudaStream_t s, std::string& err) {
  mt19937_64_kernel<<<1, 312, 0, s>>>(seed, count, dst);
  return cuda_status(err, "mt19937_64_kernel");
}

}  // namespace

int mt19937_64_device(uint64_t seed, uint64_t count, uint64_t* out, int device, std::string& err) {
  if (count > 0 && !out) {
    err = "mt19937_64: null output";
    return DBX_EINVAL;
  }
  if (cudaSetDevice(device) != cudaSuccess) return cuda_status(err, "cudaSetDevice");
  Dev D{{}, &err};
  const bool dev = on_device(out);
  uint64_t* w = dev ? out : static_cast<uint64_t*>(D.alloc(count * 8));
  if (!D.ok) return DBX_ECUDA;
  if (int st = mt_stream(seed, count, w, 0, err)) return st;
  if (!dev && cudaMemcpy(out, w, count * 8, cudaMemcpyDeviceToHost) != cudaSuccess)
    return cuda_status(err, "D2H");
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_status(err, "mt19937_64");
  return DBX_OK;
}

int gen_honest_device(int rows, int cols, int nshapes, double sinus_amp, uint64_t scene_seed, const double* taps,
                      int q1, int q2, int n1, int n2, double noise_level, uint64_t noise_seed, double* f_true,
                      double* g, int device, std::string& err) {
  if (!taps || !g || n1 < 1 || n2 < 1 || rows < n1 || cols < n2 || q1 < 0 || q2 < 0 || nshapes < 0) {
    err = "gen_honest_device: invalid argument";
    return DBX_EINVAL;
  }
  if (noise_level < 0.0) {
    err = "add_noise: negative level";  // image.hpp:73
    return DBX_EINVAL;
  }
  // experiment.hpp:76-83: centred offsets, margin >= q
  const int off1 = (rows - n1) / 2, off2 = (cols - n2) / 2;
  if (off1 < q1 || rows - off1 - n1 < q1 || off2 < q2 || cols - off2 - n2 < q2) {
    err = "synthesize: canvas margin smaller than the PSF support";
    return DBX_EINVAL;
  }
  if (cudaSetDevice(device) != cudaSuccess) return cuda_status(err, "cudaSetDevice");
  // shapes in generation order + per-tile CSR lists (host: O(shapes x tiles))
  std::vector<double> prm((size_t)nshapes * DBX_SHAPE_PARAMS);
  if (dbx_gen_scene_shapes(rows, cols, nshapes, scene_seed, prm.data()) != DBX_OK) {
    err = "gen_scene_shapes: invalid argument";
    return DBX_EINVAL;
  }
  const int tx = (cols + kTile - 1) / kTile, ty = (rows + kTile - 1) / kTile;
  std::vector<int> tstart((size_t)tx * ty + 1, 0), fill;
  for (int pass = 0; pass < 2; ++pass) {
    if (pass == 1) {
      for (size_t t = 1; t < tstart.size(); ++t) tstart[t] += tstart[t - 1];
      fill.assign(tstart.begin(), tstart.end() - 1);
    }
    std::vector<int> lists(pass ? tstart.back() : 0);
    for (int s = 0; s < nshapes; ++s) {
      const double* P = prm.data() + (size_t)s * DBX_SHAPE_PARAMS;
      const int r0 = (int)P[8], r1 = (int)P[9], c0 = (int)P[10], c1 = (int)P[11];
      if (r0 > r1 || c0 > c1) continue;
      for (int y = r0 / kTile; y <= r1 / kTile; ++y)
        for (int x = c0 / kTile; x <= c1 / kTile; ++x) {
          const size_t t = (size_t)y * tx + x;
          if (pass == 0) ++tstart[t + 1];
          else lists[fill[t]++] = s;
        }
    }
    if (pass == 1) fill.swap(lists);  // fill now holds the lists
  }
  const size_t NC = (size_t)rows * cols, N = (size_t)n1 * n2;
  Dev D{{}, &err};
  auto* dprm = static_cast<double*>(D.alloc(prm.size() * 8));
  auto* dts = static_cast<int*>(D.alloc(tstart.size() * 4));
  auto* dtl = static_cast<int*>(D.alloc(fill.size() * 4));
  auto* dscene = static_cast<double*>(D.alloc(NC * 8));
  auto* dtaps = static_cast<double*>(D.alloc((size_t)(2 * q1 + 1) * (2 * q2 + 1) * 8));
  auto* clean = static_cast<double*>(D.alloc(N * 8));
  const bool fdev = f_true && on_device(f_true), gdev = on_device(g);
  double* df = f_true ? (fdev ? f_true : static_cast<double*>(D.alloc(N * 8))) : nullptr;
  double* dg = gdev ? g : static_cast<double*>(D.alloc(N * 8));
  if (!D.ok) return DBX_ECUDA;
  cudaMemcpy(dprm, prm.data(), prm.size() * 8, cudaMemcpyHostToDevice);
  cudaMemcpy(dts, tstart.data(), tstart.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dtl, fill.data(), fill.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dtaps, taps, (size_t)(2 * q1 + 1) * (2 * q2 + 1) * 8, cudaMemcpyHostToDevice);
  if (int st = cuda_status(err, "H2D")) return st;
  paint_kernel<<<dim3(tx, ty), dim3(32, 8)>>>(dscene, rows, cols, dprm, dts, dtl, tx, sinus_amp);
  if (int st = cuda_status(err, "paint_kernel")) return st;
  const size_t hsm = ((size_t)(kHTH + 2 * q1) * (32 + 2 * q2) + (size_t)(2 * q1 + 1) * (2 * q2 + 1)) * 8;
  static AttrOnce attr;
  if (!attr.ensure(honest_kernel, hsm)) {
    err = "honest_kernel: mask too large for the staged window";
    return DBX_EINVAL;
  }
  honest_kernel<<<dim3((n2 + 31) / 32, (n1 + kHTH - 1) / kHTH), dim3(32, 8), hsm>>>(
      dscene, cols, dtaps, q1, q2, n1, n2, off1, off2, clean, df);
  if (int st = cuda_status(err, "honest_kernel")) return st;
  if (noise_level == 0.0) {
    cudaMemcpy(dg, clean, N * 8, cudaMemcpyDeviceToDevice);
  } else {
    // add_noise (image.hpp:72-82): the scene buffer is free now — words, then eta
    const uint64_t words = N + (N & 1);
    uint64_t* w = reinterpret_cast<uint64_t*>(dscene);
    double* eta = static_cast<double*>(D.alloc(N * 8));
    auto* part = static_cast<double*>(D.alloc(2 * kRedBlocks * 8 + 16));
    if (!D.ok) return DBX_ECUDA;
    if (NC < words) {
      err = "gen_honest_device: canvas smaller than the noise stream";
      return DBX_EINVAL;
    }
    if (int st = mt_stream(noise_seed, words, w, 0, err)) return st;
    box_muller_kernel<<<(unsigned)((N / 2 + 1 + 255) / 256), 256>>>(w, N, eta);
    sumsq_partial<<<kRedBlocks, 256>>>(eta, N, part);
    sum_final<<<1, 32>>>(part, kRedBlocks, part + 2 * kRedBlocks);
    sumsq_partial<<<kRedBlocks, 256>>>(clean, N, part + kRedBlocks);
    sum_final<<<1, 32>>>(part + kRedBlocks, kRedBlocks, part + 2 * kRedBlocks + 1);
    double nn[2];
    cudaMemcpy(nn, part + 2 * kRedBlocks, 16, cudaMemcpyDeviceToHost);
    if (int st = cuda_status(err, "noise")) return st;
    const double raw = std::sqrt(nn[0]);
    if (!(raw > 0.0)) {
      err = "add_noise: degenerate noise draw";
      return DBX_EINVAL;
    }
    const double s = noise_level * std::sqrt(nn[1]) / raw;
    add_scaled<<<(unsigned)((N + 255) / 256), 256>>>(clean, eta, N, s, dg);
  }
  if (int st = cuda_status(err, "add_scaled")) return st;
  if (!gdev) cudaMemcpy(g, dg, N * 8, cudaMemcpyDeviceToHost);
  if (f_true && !fdev) cudaMemcpy(f_true, df, N * 8, cudaMemcpyDeviceToHost);
  if (cudaDeviceSynchronize() != cudaSuccess) return cuda_status(err, "gen_honest_device");
  return cuda_status(err, "D2H");
}

}  // namespace dbx
