// deblur_b200.hpp — drop-in C++ face of the B200 AR-deblurring path.
//
// Re-creates the reference library's names and value semantics
// (/root/reference/proj/include/deblur/*.hpp, namespace deblur) on top of the
// C-ABI in dbx.h, for the anti-reflective preconditioned-Landweber path:
//
//   deblur::apply / apply_reblur_adjoint      blur.hpp:75-90
//   deblur::tensor_apply (SineI, AR, ARInv)   transforms.hpp:198-226
//   deblur::build_tikhonov (AR / CosineIII)   preconditioner.hpp:62-85
//   (Reflective BCs with the CosineIII algebra: SURVEY §8f f3)
//   SlabRun: d_landweber on one image in row slabs across ranks (NCCL;
//            no reference equivalent)
//   deblur::precondition_apply                preconditioner.hpp:88-90
//   deblur::landweber / d_landweber           solver.hpp:139-148
//   deblur::add_noise / rre                   image.hpp:72-91
//
// Matrix is a minimal row-major double matrix, layout-compatible with
// Eigen::Matrix<double, Dynamic, Dynamic, RowMajor> through data()/rows()/cols()
// (the reference's core.hpp:19 Matrix).  Errors map back to the reference's
// exceptions: std::invalid_argument (detail::require), SolverDivergence
// (std::runtime_error), and std::runtime_error for device failures (there is
// no CPU fallback).  Link with -ldbx (paper_1211_0393_b200/libdbx.so).
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <memory>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "dbx.h"

namespace deblur_b200 {

using Index = long;

class Matrix {
 public:
  Matrix() = default;
  Matrix(Index r, Index c, double v = 0.0) : r_(r), c_(c), a_(static_cast<size_t>(r * c), v) {}
  static Matrix Zero(Index r, Index c) { return Matrix(r, c, 0.0); }
  static Matrix Constant(Index r, Index c, double v) { return Matrix(r, c, v); }
  Index rows() const { return r_; }
  Index cols() const { return c_; }
  Index size() const { return r_ * c_; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  double& operator()(Index i, Index j) { return a_[static_cast<size_t>(i * c_ + j)]; }
  double operator()(Index i, Index j) const { return a_[static_cast<size_t>(i * c_ + j)]; }
  double norm() const {
    double s = 0.0;
    for (double v : a_) s += v * v;
    return std::sqrt(s);
  }
  double sum() const {
    double s = 0.0;
    for (double v : a_) s += v;
    return s;
  }

 private:
  Index r_ = 0, c_ = 0;
  std::vector<double> a_;
};

struct SolverDivergence : std::runtime_error {  // solver.hpp:42-44
  using std::runtime_error::runtime_error;
};

namespace detail {
inline void check(int st) {
  if (st == DBX_OK) return;
  const std::string msg = dbx_last_error();
  if (st == DBX_EINVAL) throw std::invalid_argument(msg);
  if (st == DBX_EDIVERGED) throw SolverDivergence(msg);
  throw std::runtime_error(msg);
}
inline void require(bool c, const std::string& what) {  // core.hpp:26-28
  if (!c) throw std::invalid_argument(what);
}
struct PlanDeleter {
  void operator()(dbx_plan* p) const { dbx_plan_destroy(p); }
};
using PlanPtr = std::shared_ptr<dbx_plan>;
inline PlanPtr make_plan(Index n1, Index n2, const Matrix& taps, Index q1, Index q2,
                         int bc = DBX_BC_ANTIREFLECTIVE) {
  dbx_plan* p = nullptr;
  check(dbx_plan_create(static_cast<int>(n1), static_cast<int>(n2), 1, taps.data(), static_cast<int>(q1),
                        static_cast<int>(q2), bc, 0, &p));
  return PlanPtr(p, PlanDeleter{});
}
// One identity-mask transform plan per (shape, BC) and thread: a hot loop of
// tensor_apply calls reuses its device buffers and DST/DCT tables instead of
// allocating a plan per call (plans are per-stream, so per thread).
inline dbx_plan* transform_plan(Index n1, Index n2, int bc) {
  thread_local std::map<std::pair<std::pair<Index, Index>, int>, PlanPtr> cache;
  auto& slot = cache[{{n1, n2}, bc}];
  if (!slot) {
    Matrix one = Matrix::Zero(1, 1);
    one(0, 0) = 1.0;
    slot = make_plan(n1, n2, one, 0, 0, bc);
  }
  return slot.get();
}
}  // namespace detail

// psf.hpp:13-39
class Psf {
 public:
  explicit Psf(Matrix taps) : taps_(std::move(taps)) {
    detail::require(taps_.rows() >= 1 && taps_.cols() >= 1 && taps_.rows() % 2 == 1 && taps_.cols() % 2 == 1,
                    "Psf: taps must have odd dimensions");
    for (Index i = 0; i < taps_.rows(); ++i)
      for (Index j = 0; j < taps_.cols(); ++j) {
        detail::require(std::isfinite(taps_(i, j)), "Psf: taps must be finite");
        detail::require(taps_(i, j) >= 0.0, "Psf: taps must be nonnegative");
      }
    detail::require(std::abs(taps_.sum() - 1.0) <= kMassTol, "Psf: taps must sum to 1 (within 1e-12)");
    q1_ = (taps_.rows() - 1) / 2;
    q2_ = (taps_.cols() - 1) / 2;
  }
  Index q1() const { return q1_; }
  Index q2() const { return q2_; }
  const Matrix& taps() const { return taps_; }
  double tap(Index i1, Index i2) const { return taps_(q1_ + i1, q2_ + i2); }
  static constexpr double kMassTol = 1e-12;

 private:
  Matrix taps_;
  Index q1_ = 0, q2_ = 0;
};

inline Psf delta_psf(Index q1 = 0, Index q2 = 0) {  // psf.hpp:41-46
  Matrix t = Matrix::Zero(2 * q1 + 1, 2 * q2 + 1);
  t(q1, q2) = 1.0;
  return Psf(std::move(t));
}

enum class BoundaryCondition { Zero, Periodic, Reflective, AntiReflective };  // boundary.hpp:9
enum class TransformKind { Dft, CosineIII, SineI, AntiReflective, AntiReflectiveInverse };  // transforms.hpp:17
enum class Algebra { Circulant, CosineIII, Tau, AntiReflective };  // spectral.hpp:12

// blur.hpp:17-34 — the device plan is created once and shared by copies.
class BlurOperator {
 public:
  BlurOperator(Psf psf, BoundaryCondition bc, Index n1, Index n2)
      : psf_(std::move(psf)), bc_(bc), n1_(n1), n2_(n2) {
    detail::require(n1 >= 1 && n2 >= 1, "BlurOperator: empty field of view");
    detail::require(bc == BoundaryCondition::AntiReflective || bc == BoundaryCondition::Reflective,
                    "BlurOperator: the B200 path implements AntiReflective and Reflective BCs");
    plan_ = detail::make_plan(n1, n2, psf_.taps(), psf_.q1(), psf_.q2(),
                              bc == BoundaryCondition::Reflective ? DBX_BC_REFLECTIVE : DBX_BC_ANTIREFLECTIVE);
  }
  const Psf& psf() const { return psf_; }
  BoundaryCondition bc() const { return bc_; }
  Index n1() const { return n1_; }
  Index n2() const { return n2_; }
  dbx_plan* plan() const { return plan_.get(); }

 private:
  Psf psf_;
  BoundaryCondition bc_;
  Index n1_, n2_;
  detail::PlanPtr plan_;
};

inline Matrix apply(const BlurOperator& op, const Matrix& f) {  // blur.hpp:75-83
  detail::require(f.rows() == op.n1() && f.cols() == op.n2(),
                  "apply: image does not match the operator's field of view");
  Matrix y(f.rows(), f.cols());
  detail::check(dbx_blur_apply(op.plan(), f.data(), y.data(), 0));
  return y;
}

inline Matrix apply_reblur_adjoint(const BlurOperator& op, const Matrix& r) {  // blur.hpp:87-90
  detail::require(r.rows() == op.n1() && r.cols() == op.n2(),
                  "apply: image does not match the operator's field of view");
  Matrix y(r.rows(), r.cols());
  detail::check(dbx_blur_apply(op.plan(), r.data(), y.data(), 1));
  return y;
}

inline Matrix tensor_apply(TransformKind kind, const Matrix& x) {  // transforms.hpp:198-226
  detail::require(kind != TransformKind::Dft, "tensor_apply: Dft is complex, use dft2_forward");
  const int bc = kind == TransformKind::CosineIII ? DBX_BC_REFLECTIVE : DBX_BC_ANTIREFLECTIVE;
  Matrix y(x.rows(), x.cols());
  detail::check(dbx_tensor_apply(detail::transform_plan(x.rows(), x.cols(), bc), static_cast<int>(kind), x.data(),
                                 y.data()));
  return y;
}

struct PreconditionerSpec {  // preconditioner.hpp:17-20
  Algebra algebra = Algebra::AntiReflective;
  double alpha = 0.0;
};

struct FilteredOperator {  // preconditioner.hpp:24-28
  Algebra algebra = Algebra::AntiReflective;
  Matrix eigs;  // d_j grid (sop.eigs)
  std::optional<Psf> source_psf;
  double alpha = 0.0;
  Index n1 = 0, n2 = 0;
  detail::PlanPtr plan;
};

inline Psf symmetrize(const Psf& p) {  // psf.hpp:71-85
  const Index q1 = p.q1(), q2 = p.q2();
  Matrix s(2 * q1 + 1, 2 * q2 + 1);
  for (Index i1 = 0; i1 <= q1; ++i1)
    for (Index i2 = 0; i2 <= q2; ++i2) {
      const double avg = (p.tap(-i1, -i2) + p.tap(-i1, i2) + p.tap(i1, -i2) + p.tap(i1, i2)) / 4.0;
      s(q1 + i1, q2 + i2) = avg;
      s(q1 - i1, q2 + i2) = avg;
      s(q1 + i1, q2 - i2) = avg;
      s(q1 - i1, q2 - i2) = avg;
    }
  return Psf(std::move(s));
}

inline FilteredOperator build_tikhonov(const Psf& p, const PreconditionerSpec& spec, Index n1, Index n2) {
  detail::require(spec.algebra == Algebra::AntiReflective || spec.algebra == Algebra::CosineIII,
                  "build_tikhonov: the B200 path implements the AntiReflective and CosineIII algebras");
  FilteredOperator d;
  d.plan = detail::make_plan(n1, n2, p.taps(), p.q1(), p.q2(),
                             spec.algebra == Algebra::CosineIII ? DBX_BC_REFLECTIVE : DBX_BC_ANTIREFLECTIVE);
  d.algebra = spec.algebra;
  detail::check(dbx_precond_build(d.plan.get(), spec.alpha));
  d.eigs = Matrix(n1, n2);
  detail::check(dbx_precond_eigs(d.plan.get(), d.eigs.data()));
  d.source_psf = symmetrize(p);
  d.alpha = spec.alpha;
  d.n1 = n1;
  d.n2 = n2;
  return d;
}

inline Matrix precondition_apply(const FilteredOperator& d, const Matrix& r) {  // preconditioner.hpp:88-90
  detail::require(r.rows() == d.n1 && r.cols() == d.n2, "filter_apply: size mismatch");
  Matrix y(r.rows(), r.cols());
  detail::check(dbx_precond_apply(d.plan.get(), r.data(), y.data()));
  return y;
}

struct StoppingRule {  // solver.hpp:17-32
  enum class Kind { FixedIterations, MinRre, RelativeResidualBelow };
  Kind kind = Kind::MinRre;
  int fixed_iterations = 0;
  double residual_threshold = 0.0;
  static StoppingRule fixed(int k) {
    detail::require(k >= 0, "StoppingRule: negative iteration count");
    return {Kind::FixedIterations, k, 0.0};
  }
  static StoppingRule min_rre() { return {Kind::MinRre, 0, 0.0}; }
  static StoppingRule residual_below(double eps) {
    detail::require(eps > 0.0, "StoppingRule: threshold must be positive");
    return {Kind::RelativeResidualBelow, 0, eps};
  }
};

struct SolverConfig {  // solver.hpp:34-39
  double tau = 1.0;
  int max_iters = 100;
  StoppingRule stop = StoppingRule::min_rre();
  std::optional<Matrix> track_rre_against;
};

struct RestorationRun {  // solver.hpp:46-52
  Matrix restored;
  int iterations_executed = 0;
  int best_iteration = 0;
  std::vector<double> rre_history;
  std::vector<double> residual_history;
};

namespace detail {
inline RestorationRun run(const BlurOperator& op, const FilteredOperator* d, const Matrix& g,
                          const SolverConfig& cfg, bool cg = false) {
  require(g.rows() == op.n1() && g.cols() == op.n2(), "landweber: data size mismatch");
  if (cfg.track_rre_against)
    require(cfg.track_rre_against->rows() == g.rows() && cfg.track_rre_against->cols() == g.cols(),
            "landweber: true image size mismatch");
  if (d) {
    require(d->n1 == op.n1() && d->n2 == op.n2(), "d_landweber: preconditioner size mismatch");
    require((d->algebra == Algebra::CosineIII) == (op.bc() == BoundaryCondition::Reflective),
            "d_landweber: the preconditioner's algebra does not match the operator's boundary condition");
    check(dbx_precond_set_eigs(op.plan(), d->eigs.data()));
  }
  const int total = cfg.stop.kind == StoppingRule::Kind::FixedIterations ? cfg.stop.fixed_iterations
                                                                        : cfg.max_iters;
  const size_t H = static_cast<size_t>(total > 0 ? total : 1);
  std::vector<double> rre(H), res(H);
  int best = 0, done = 0;
  RestorationRun out;
  out.restored = Matrix(g.rows(), g.cols());
  const double* f = cfg.track_rre_against ? cfg.track_rre_against->data() : nullptr;
  if (cg)
    check(dbx_cgls_run(op.plan(), g.data(), f, cfg.max_iters, static_cast<int>(cfg.stop.kind),
                       cfg.stop.fixed_iterations, cfg.stop.residual_threshold, d ? 1 : 0, out.restored.data(),
                       rre.data(), res.data(), &best, &done, nullptr));
  else
    check(dbx_landweber_run(op.plan(), g.data(), f, cfg.tau, cfg.max_iters, static_cast<int>(cfg.stop.kind),
                            cfg.stop.fixed_iterations, cfg.stop.residual_threshold, d ? 1 : 0,
                            out.restored.data(), rre.data(), res.data(), &best, &done, nullptr));
  out.iterations_executed = done;
  out.best_iteration = best;
  out.residual_history.assign(res.begin(), res.begin() + done);
  if (f) out.rre_history.assign(rre.begin(), rre.begin() + done);
  return out;
}
}  // namespace detail

inline RestorationRun landweber(const BlurOperator& op, const Matrix& g, const SolverConfig& cfg) {
  return detail::run(op, nullptr, g, cfg);  // solver.hpp:139-142
}

inline RestorationRun d_landweber(const BlurOperator& op, const FilteredOperator& d, const Matrix& g,
                                  const SolverConfig& cfg) {
  return detail::run(op, &d, g, cfg);  // solver.hpp:145-148
}

// Reblurred CGLS, plain (d == nullptr) or preconditioned (no
// reference equivalent).
inline RestorationRun cgls(const BlurOperator& op, const Matrix& g, const SolverConfig& cfg,
                           const FilteredOperator* d = nullptr) {
  return detail::run(op, d, g, cfg, true);
}

struct SemiconvergenceReport {  // solver.hpp:150-151
  int best_iter = 0;       // 1-based
  double best_rre = 0.0;
  bool diverged_after = false;
};

// First RRE minimum (std::min_element) and whether the last RRE degrades by
// more than 5% past it (solver.hpp:152-160).  Host-side post-process.
inline SemiconvergenceReport semiconvergence_report(const RestorationRun& run) {
  detail::require(!run.rre_history.empty(), "semiconvergence_report: no RRE history");
  std::size_t b = 0;
  for (std::size_t i = 1; i < run.rre_history.size(); ++i)
    if (run.rre_history[i] < run.rre_history[b]) b = i;
  SemiconvergenceReport rep;
  rep.best_iter = static_cast<int>(b) + 1;
  rep.best_rre = run.rre_history[b];
  rep.diverged_after = run.rre_history.back() > rep.best_rre * 1.05;
  return rep;
}

// d_landweber on one n x n image split into row slabs across ranks (C++
// loop behind dbx_slab_run: NCCL halos, all-to-all from grouped send/recv,
// device all-reduce and bookkeeping).  rank >= 0 with a communicator (the
// caller's ncclComm_t via dbx_comm_wrap, or dbx_comm_init); rank = -1 holds
// all slabs in this process.  g, f, x_out: DEVICE arrays of the rows held here.
class SlabRun {
 public:
  SlabRun(Index n, int parts, int rank, const Psf& psf, double alpha, dbx_comm* comm = nullptr, int device = 0) {
    detail::require(psf.q1() == psf.q2(), "SlabRun: square masks only (one q for both axes)");
    dbx_slab* s = nullptr;
    detail::check(dbx_slab_create(static_cast<int>(n), parts, rank, psf.taps().data(), static_cast<int>(psf.q1()),
                                  static_cast<int>(psf.q2()), alpha, comm, device, &s));
    slab_.reset(s);
  }
  // returns the histories; x_out receives the restored rows (best-RRE iterate
  // when f is given, solver.hpp:127-131)
  RestorationRun run(const double* g, const double* f, double* x_out, const SolverConfig& cfg) {
    const int total = cfg.stop.kind == StoppingRule::Kind::FixedIterations ? cfg.stop.fixed_iterations
                                                                          : cfg.max_iters;
    detail::require(total >= 1, "SolverConfig: max_iters must be >= 1");
    std::vector<double> rre(static_cast<size_t>(total)), res(static_cast<size_t>(total));
    int best = 0, done = 0;
    detail::check(dbx_slab_run(slab_.get(), g, f, cfg.tau, total, static_cast<int>(cfg.stop.kind),
                               cfg.stop.residual_threshold, x_out, rre.data(), res.data(), &best, &done));
    RestorationRun out;
    out.iterations_executed = done;
    out.best_iteration = best;
    out.residual_history.assign(res.begin(), res.begin() + done);
    if (f) out.rre_history.assign(rre.begin(), rre.begin() + done);
    return out;
  }

 private:
  struct Del {
    void operator()(dbx_slab* s) const { dbx_slab_destroy(s); }
  };
  std::unique_ptr<dbx_slab, Del> slab_;
};

struct NoiseSpec {  // image.hpp:31-34
  double relative_level = 0.0;
  std::uint64_t seed = 0;
};

inline Matrix add_noise(const Matrix& g, const NoiseSpec& spec) {  // image.hpp:72-82
  Matrix out(g.rows(), g.cols());
  detail::check(dbx_add_noise(g.data(), static_cast<int>(g.rows()), static_cast<int>(g.cols()),
                              spec.relative_level, spec.seed, out.data()));
  return out;
}

inline double rre(const Matrix& x, const Matrix& f) {  // image.hpp:85-91
  detail::require(x.rows() == f.rows() && x.cols() == f.cols(), "rre: dimension mismatch");
  const double den = f.norm();
  detail::require(den > 0.0, "rre: zero true image");
  double s = 0.0;
  for (Index i = 0; i < x.rows(); ++i)
    for (Index j = 0; j < x.cols(); ++j) s += (x(i, j) - f(i, j)) * (x(i, j) - f(i, j));
  return std::sqrt(s) / den;
}

}  // namespace deblur_b200
