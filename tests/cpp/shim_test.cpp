// Exercises include/deblur_b200.hpp (the C++ drop-in face) end to end on the
// GPU with known answers from the reference tests; prints "OK" on success.
#include <cuda_runtime.h>

#include <cstdio>
#include <random>

#include "deblur_b200.hpp"

using namespace deblur_b200;

#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::fprintf(stderr, "FAILED %s:%d %s\n", __FILE__, __LINE__, #c); \
      return 1;                                                    \
    }                                                              \
  } while (0)

int main() {
  if (dbx_device_count() < 1) {
    std::printf("NO_DEVICE\n");
    return 2;
  }
  std::mt19937_64 rng(43);
  std::uniform_real_distribution<double> u(0.05, 1.0);
  // constant images are fixed points (blur_test.cpp:21-31)
  Matrix t(5, 3);
  for (Index i = 0; i < 5; ++i)
    for (Index j = 0; j < 3; ++j) t(i, j) = u(rng);
  const double s = t.sum();
  for (Index i = 0; i < 5; ++i)
    for (Index j = 0; j < 3; ++j) t(i, j) /= s;
  BlurOperator op(Psf(t), BoundaryCondition::AntiReflective, 7, 7);
  Matrix c = Matrix::Constant(7, 7, 4.5);
  Matrix g = apply(op, c);
  for (Index i = 0; i < 7; ++i)
    for (Index j = 0; j < 7; ++j) CHECK(std::abs(g(i, j) - 4.5) <= 1e-13);
  // D-Landweber with a delta mask: x1 = g/(1+alpha) (solver_test.cpp:133-150)
  Matrix gg(8, 8);
  for (Index i = 0; i < 8; ++i)
    for (Index j = 0; j < 8; ++j) gg(i, j) = 1.0 + u(rng);
  BlurOperator dop(delta_psf(), BoundaryCondition::AntiReflective, 8, 8);
  auto d = build_tikhonov(delta_psf(), {Algebra::AntiReflective, 0.25}, 8, 8);
  SolverConfig cfg;
  cfg.stop = StoppingRule::fixed(1);
  cfg.max_iters = 1;
  auto run = d_landweber(dop, d, gg, cfg);
  for (Index i = 0; i < 8; ++i)
    for (Index j = 0; j < 8; ++j) CHECK(std::abs(run.restored(i, j) - gg(i, j) / 1.25) <= 1e-12);
  // semiconvergence_report (solver.hpp:152-160): first minimum, 5% rule
  {
    RestorationRun h;
    h.rre_history = {0.5, 0.3, 0.2, 0.2, 0.25};
    auto rep = semiconvergence_report(h);
    CHECK(rep.best_iter == 3 && rep.best_rre == 0.2 && rep.diverged_after);
    h.rre_history = {0.5, 0.3, 0.2, 0.2, 0.205};
    CHECK(!semiconvergence_report(h).diverged_after);
    bool empty_threw = false;
    try {
      semiconvergence_report(RestorationRun{});
    } catch (const std::invalid_argument&) {
      empty_threw = true;
    }
    CHECK(empty_threw);
  }
  // errors map to the reference exceptions
  bool threw = false;
  try {
    apply(op, Matrix(7, 8));
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    SolverConfig bad;
    bad.tau = 3.0;
    bad.max_iters = 200;
    bad.stop = StoppingRule::fixed(200);
    BlurOperator id(delta_psf(1, 1), BoundaryCondition::AntiReflective, 8, 8);
    landweber(id, gg, bad);
  } catch (const SolverDivergence&) {
    threw = true;
  }
  CHECK(threw);
  // T T~ = I through tensor_apply
  Matrix x(9, 11);
  for (Index i = 0; i < 9; ++i)
    for (Index j = 0; j < 11; ++j) x(i, j) = u(rng);
  Matrix back = tensor_apply(TransformKind::AntiReflective, tensor_apply(TransformKind::AntiReflectiveInverse, x));
  for (Index i = 0; i < 9; ++i)
    for (Index j = 0; j < 11; ++j) CHECK(std::abs(back(i, j) - x(i, j)) <= 1e-12);
  // R R^T = I through the cached CosineIII plan (reflective algebra)
  {
    Matrix rb = tensor_apply(TransformKind::CosineIII, x);
    Matrix xx(9, 11);
    for (int rep = 0; rep < 3; ++rep) xx = tensor_apply(TransformKind::AntiReflective, tensor_apply(TransformKind::AntiReflectiveInverse, x));
    CHECK(std::abs(xx(4, 5) - x(4, 5)) <= 1e-12);
    CHECK(rb.rows() == 9 && rb.cols() == 11);
  }
  // Reflective BCs: constants are fixed points; the CosineIII preconditioner of a
  // delta mask gives x1 = g / (1 + alpha); mixing algebra and BC is refused
  {
    BlurOperator rop(Psf(t), BoundaryCondition::Reflective, 7, 7);
    Matrix rg = apply(rop, c);
    for (Index i = 0; i < 7; ++i)
      for (Index j = 0; j < 7; ++j) CHECK(std::abs(rg(i, j) - 4.5) <= 1e-13);
    BlurOperator rdop(delta_psf(), BoundaryCondition::Reflective, 8, 8);
    auto rd = build_tikhonov(delta_psf(), {Algebra::CosineIII, 0.25}, 8, 8);
    auto rrun = d_landweber(rdop, rd, gg, cfg);
    for (Index i = 0; i < 8; ++i)
      for (Index j = 0; j < 8; ++j) CHECK(std::abs(rrun.restored(i, j) - gg(i, j) / 1.25) <= 1e-12);
    bool mix = false;
    try {
      d_landweber(dop, rd, gg, cfg);
    } catch (const std::invalid_argument&) {
      mix = true;
    }
    CHECK(mix);
  }
  // C++ row-slab loop (2 in-process slabs) == the single-image D-Landweber
  {
    const Index n = 32;
    Matrix m(5, 5);
    for (Index i = 0; i < 5; ++i)
      for (Index j = 0; j < 5; ++j) m(i, j) = u(rng);
    const double ms = m.sum();
    for (Index i = 0; i < 5; ++i)
      for (Index j = 0; j < 5; ++j) m(i, j) /= ms;
    Psf mp(m);
    Matrix f0(n, n), g0(n, n);
    for (Index i = 0; i < n; ++i)
      for (Index j = 0; j < n; ++j) f0(i, j) = u(rng);
    BlurOperator sop(mp, BoundaryCondition::AntiReflective, n, n);
    g0 = apply(sop, f0);
    auto sd = build_tikhonov(mp, {Algebra::AntiReflective, 0.05}, n, n);
    SolverConfig scfg;
    scfg.max_iters = 6;
    scfg.track_rre_against = f0;
    auto ref = d_landweber(sop, sd, g0, scfg);
    const size_t bytes = sizeof(double) * n * n;
    double *dg = nullptr, *df = nullptr, *dx = nullptr;
    CHECK(cudaMalloc(&dg, bytes) == cudaSuccess && cudaMalloc(&df, bytes) == cudaSuccess &&
          cudaMalloc(&dx, bytes) == cudaSuccess);
    cudaMemcpy(dg, g0.data(), bytes, cudaMemcpyHostToDevice);
    cudaMemcpy(df, f0.data(), bytes, cudaMemcpyHostToDevice);
    SlabRun slabs(n, 2, -1, mp, 0.05);
    auto srun = slabs.run(dg, df, dx, scfg);
    Matrix xs(n, n);
    cudaMemcpy(xs.data(), dx, bytes, cudaMemcpyDeviceToHost);
    cudaFree(dg);
    cudaFree(df);
    cudaFree(dx);
    CHECK(srun.best_iteration == ref.best_iteration && srun.iterations_executed == ref.iterations_executed);
    double e = 0.0, nr = 0.0;
    for (Index i = 0; i < n; ++i)
      for (Index j = 0; j < n; ++j) {
        e += (xs(i, j) - ref.restored(i, j)) * (xs(i, j) - ref.restored(i, j));
        nr += ref.restored(i, j) * ref.restored(i, j);
      }
    CHECK(std::sqrt(e / nr) <= 1e-10);
    for (size_t k = 0; k < ref.rre_history.size(); ++k)
      CHECK(std::abs(srun.rre_history[k] - ref.rre_history[k]) <= 1e-10 * ref.rre_history[k]);
  }
  std::printf("OK\n");
  return 0;
}
