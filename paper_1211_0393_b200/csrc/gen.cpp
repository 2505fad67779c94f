// gen.cpp — host-side synthetic input generation for the BASELINE configs
// (scene, masks, Honest blur-then-crop, add_noise).  Inputs are produced once
// on the host so the GPU path and the CPU oracle consume bit-identical data.
// Not on the timed path.
//
// Restated reference pieces: add_noise + GaussianSampler (image.hpp:44-82,
// bit-exact: std::mt19937_64 is fully specified by the C++ standard),
// synthesize Honest branch (experiment.hpp:71-99), Gaussian mask sampling
// (psf.hpp:126-138, generalised to anisotropic / rotated).  The scene and
// motion-mask generators are new (the reference scene is an analytic ramp,
// synthetic.hpp:15-40); their definitions are recorded in DESIGN.md.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <thread>
#include <vector>

#include "../../include/dbx.h"

namespace {

constexpr double kPi = 3.141592653589793238462643383279502884;

thread_local std::string g_gen_err;

// U[0,1) from the top 53 bits (implementation-independent, unlike
// std::uniform_real_distribution).
inline double u01(std::mt19937_64& r) { return double(r() >> 11) * 0x1p-53; }

double fro(const double* x, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += x[i] * x[i];
  return std::sqrt(s);
}

// image.hpp:44-66
struct GaussianSampler {
  std::mt19937_64 rng;
  double spare = 0.0;
  bool have = false;
  explicit GaussianSampler(uint64_t s) : rng(s) {}
  double operator()() {
    if (have) {
      have = false;
      return spare;
    }
    const double u1 = (double(rng() >> 11) + 1.0) * 0x1p-53;
    const double u2 = double(rng() >> 11) * 0x1p-53;
    const double r = std::sqrt(-2.0 * std::log(u1));
    const double a = 2.0 * kPi * u2;
    spare = r * std::sin(a);
    have = true;
    return r * std::cos(a);
  }
};

int normalise(double* t, size_t n) {
  double s = 0.0;
  for (size_t i = 0; i < n; ++i) s += t[i];
  if (!(s > 0.0)) return DBX_EINVAL;
  for (size_t i = 0; i < n; ++i) t[i] /= s;  // t /= t.sum() (psf.hpp:136)
  return DBX_OK;
}

}  // namespace

extern "C" {

int dbx_add_noise(const double* g, int n1, int n2, double level, uint64_t seed, double* out) {
  if (level < 0.0) return DBX_EINVAL;  // image.hpp:73
  const size_t n = (size_t)n1 * (size_t)n2;
  if (level == 0.0) {
    if (out != g) std::memcpy(out, g, n * sizeof(double));
    return DBX_OK;
  }
  GaussianSampler gs(seed);
  std::vector<double> eta(n);
  for (size_t i = 0; i < n; ++i) eta[i] = gs();  // row-major fill (image.hpp:76-77)
  const double raw = fro(eta.data(), n);
  if (!(raw > 0.0)) return DBX_EINVAL;
  const double s = level * fro(g, n) / raw;
  for (size_t i = 0; i < n; ++i) out[i] = g[i] + s * eta[i];
  return DBX_OK;
}

int dbx_gen_scene_shapes(int rows, int cols, int nshapes, uint64_t seed, double* params) {
  if (rows < 1 || cols < 1 || nshapes < 0 || (nshapes > 0 && !params)) return DBX_EINVAL;
  std::mt19937_64 rng(seed);
  const double dim = std::min(rows, cols);
  for (int s = 0; s < nshapes; ++s) {
    double* P = params + (size_t)s * DBX_SHAPE_PARAMS;
    const bool ellipse = u01(rng) < 0.5;
    const double cy = u01(rng) * rows, cx = u01(rng) * cols;
    const double a = (0.02 + 0.10 * u01(rng)) * dim;
    const double b = (0.02 + 0.10 * u01(rng)) * dim;
    const double th = u01(rng) * kPi;
    const double val = u01(rng);
    const double rad = std::max(a, b) * (ellipse ? 1.0 : std::sqrt(2.0));
    P[0] = ellipse ? 1.0 : 0.0; P[1] = cy; P[2] = cx; P[3] = a; P[4] = b;
    P[5] = std::cos(th); P[6] = std::sin(th); P[7] = val;
    // clipped bounding box (rows r0..r1, cols c0..c1): the only pixels tested
    P[8] = std::max(0, (int)std::floor(cy - rad)); P[9] = std::min(rows - 1, (int)std::ceil(cy + rad));
    P[10] = std::max(0, (int)std::floor(cx - rad)); P[11] = std::min(cols - 1, (int)std::ceil(cx + rad));
  }
  return DBX_OK;
}

int dbx_gen_scene(int rows, int cols, int nshapes, double sinus_amp, uint64_t seed, double* out) {
  if (rows < 1 || cols < 1 || nshapes < 0 || !out) return DBX_EINVAL;
  std::vector<double> prm((size_t)nshapes * DBX_SHAPE_PARAMS);
  if (dbx_gen_scene_shapes(rows, cols, nshapes, seed, prm.data()) != DBX_OK) return DBX_EINVAL;
  std::fill(out, out + (size_t)rows * cols, 0.0);
  for (int s = 0; s < nshapes; ++s) {
    const double* P = prm.data() + (size_t)s * DBX_SHAPE_PARAMS;
    const bool ellipse = P[0] != 0.0;
    const double cy = P[1], cx = P[2], a = P[3], b = P[4], ct = P[5], st = P[6], val = P[7];
    const int r0 = (int)P[8], r1 = (int)P[9], c0 = (int)P[10], c1 = (int)P[11];
    for (int r = r0; r <= r1; ++r) {
      const double dy = r + 0.5 - cy;
      double* row = out + (size_t)r * cols;
      for (int c = c0; c <= c1; ++c) {
        // gen.cpp is compiled with -ffp-contract=off: the same IEEE operations
        // as the device painter (gen_dev.cu), so both make identical in/out calls
        const double dx = c + 0.5 - cx;
        const double u = dx * ct + dy * st, v = -dx * st + dy * ct;
        const bool in = ellipse ? (u * u) / (a * a) + (v * v) / (b * b) <= 1.0
                                : std::fabs(u) <= a && std::fabs(v) <= b;
        if (in) row[c] = val;  // painter's rule: later shapes overwrite
      }
    }
  }
  if (sinus_amp != 0.0)
    for (int r = 0; r < rows; ++r)
      for (int c = 0; c < cols; ++c)
        out[(size_t)r * cols + c] +=
            sinus_amp * std::sin(2.0 * kPi * (3.0 * (r + 0.5) / rows + 2.0 * (c + 0.5) / cols));
  return DBX_OK;
}

int dbx_mt19937_64_host(uint64_t seed, uint64_t count, uint64_t* out) {
  if (count > 0 && !out) return DBX_EINVAL;
  std::mt19937_64 rng(seed);
  for (uint64_t i = 0; i < count; ++i) out[i] = rng();
  return DBX_OK;
}

int dbx_gen_psf_gaussian(int q1, int q2, double sigma1, double sigma2, double theta_deg,
                         double off1, double off2, double* taps) {
  if (q1 < 0 || q2 < 0 || !(sigma1 > 0.0) || !(sigma2 > 0.0) || !taps) return DBX_EINVAL;
  const double th = theta_deg * kPi / 180.0, ct = std::cos(th), st = std::sin(th);
  const int W = 2 * q2 + 1;
  for (int i1 = -q1; i1 <= q1; ++i1)
    for (int i2 = -q2; i2 <= q2; ++i2) {
      const double d1 = (double)i1 - off1, d2 = (double)i2 - off2;  // (row, col)
      const double u = ct * d1 + st * d2, v = -st * d1 + ct * d2;
      taps[(size_t)(q1 + i1) * W + (q2 + i2)] =
          std::exp(-0.5 * (u * u / (sigma1 * sigma1) + v * v / (sigma2 * sigma2)));
    }
  return normalise(taps, (size_t)(2 * q1 + 1) * W);
}

int dbx_gen_psf_motion(int q1, int q2, double length, double angle_deg, double tail, double* taps) {
  if (q1 < 0 || q2 < 0 || !(length > 0.0) || !(tail > 0.0) || !taps) return DBX_EINVAL;
  const int H = 2 * q1 + 1, W = 2 * q2 + 1;
  std::fill(taps, taps + (size_t)H * W, 0.0);
  const double a = angle_deg * kPi / 180.0;
  // direction in (row, col): rows grow downwards, angle counter-clockwise from +col
  const double dr = -std::sin(a), dc = std::cos(a);
  const double half = 0.5 * length;
  const int per_px = 64;
  const double smax = 4.0 * std::max(q1, q2) + length;
  for (long i = 0;; ++i) {
    const double s = -half + (double)i / per_px;
    if (s > smax) break;
    const double w = s <= half ? 1.0 : std::exp(-(s - half) / tail);  // one-sided tail
    const double pr = q1 + s * dr, pc = q2 + s * dc;
    const int r0 = (int)std::floor(pr), c0 = (int)std::floor(pc);
    const double fr = pr - r0, fc = pc - c0;
    const double wts[4] = {(1 - fr) * (1 - fc), (1 - fr) * fc, fr * (1 - fc), fr * fc};
    const int rr[4] = {r0, r0, r0 + 1, r0 + 1}, cc[4] = {c0, c0 + 1, c0, c0 + 1};
    for (int k = 0; k < 4; ++k)
      if (rr[k] >= 0 && rr[k] < H && cc[k] >= 0 && cc[k] < W) taps[(size_t)rr[k] * W + cc[k]] += w * wts[k];
  }
  return normalise(taps, (size_t)H * W);
}

int dbx_gen_honest(const double* scene, int rows, int cols, const double* taps, int q1, int q2,
                   int n1, int n2, double noise_level, uint64_t noise_seed, int threads,
                   double* f_true, double* g) {
  if (!scene || !taps || !g || n1 < 1 || n2 < 1 || rows < n1 || cols < n2) return DBX_EINVAL;
  // experiment.hpp:76-83: centred offsets, margin >= q
  const int off1 = (rows - n1) / 2, off2 = (cols - n2) / 2;
  if (off1 < q1 || rows - off1 - n1 < q1 || off2 < q2 || cols - off2 - n2 < q2) return DBX_EINVAL;
  if (f_true)
    for (int r = 0; r < n1; ++r)
      std::memcpy(f_true + (size_t)r * n2, scene + (size_t)(off1 + r) * cols + off2, n2 * sizeof(double));
  const int W = 2 * q2 + 1;
  std::vector<double> clean((size_t)n1 * n2);
  // experiment.hpp:85-92: g(r,c) = sum_s h_s scene(off + r - s)
  auto work = [&](int rbeg, int rend) {
    for (int r = rbeg; r < rend; ++r)
      for (int c = 0; c < n2; ++c) {
        double acc = 0.0;
        for (int s1 = -q1; s1 <= q1; ++s1) {
          const double* srow = scene + (size_t)(off1 + r - s1) * cols + (off2 + c);
          const double* trow = taps + (size_t)(q1 + s1) * W + q2;
          for (int s2 = -q2; s2 <= q2; ++s2) acc += trow[s2] * srow[-s2];
        }
        clean[(size_t)r * n2 + c] = acc;
      }
  };
  int nt = threads > 0 ? threads : (int)std::max(1u, std::thread::hardware_concurrency());
  nt = std::min(nt, n1);
  std::vector<std::thread> pool;
  for (int t = 0; t < nt; ++t) pool.emplace_back(work, (int)((long)n1 * t / nt), (int)((long)n1 * (t + 1) / nt));
  for (auto& th : pool) th.join();
  return dbx_add_noise(clean.data(), n1, n2, noise_level, noise_seed, g);
}

}  // extern "C"
