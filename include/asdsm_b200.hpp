// asdsm_b200.hpp -- header-only C++17 mirror of the reference's public solver API
// (proj/include/asdsm/{mesh,problems,solver,errors}.hpp of arxiv/paper_2303_01163) over the
// C-ABI of libasdsm_b200.so (asdsm_b200.h).  Same names, argument meanings and exception
// classes, so a caller of asdsm::asdsm_iterate / asdsm::SolverContext switches by changing the
// namespace:
//
//   auto problem = asdsm_b200::make_problem(1, 1);
//   auto mesh = asdsm_b200::example_mesh(1, 1, 1029, 9);
//   asdsm_b200::IterationState st = asdsm_b200::asdsm_iterate(problem, mesh, {});
//
// Host vectors in and out (the reference's GridFunction::values); the device-resident entry
// points (asdsm_iterate_async, asdsm_device_solution) are reachable through SolverContext::plan().
// Link: -I include -L paper_2303_01163_b200 -lasdsm_b200.
#pragma once

#include <cstdint>
#include <functional>
#include <array>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "asdsm_b200.h"

namespace asdsm_b200 {

// ---- errors (errors.hpp:8-66) -----------------------------------------------------------
struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
#define ASDSM_B200_ERROR_CLASS(NAME) \
  struct NAME : Error {              \
    using Error::Error;              \
  };
ASDSM_B200_ERROR_CLASS(DivisibilityError)
ASDSM_B200_ERROR_CLASS(DegenerateError)
ASDSM_B200_ERROR_CLASS(IndexOutOfRange)
ASDSM_B200_ERROR_CLASS(NotASubmesh)
ASDSM_B200_ERROR_CLASS(InvalidKind)
ASDSM_B200_ERROR_CLASS(DimensionMismatch)
ASDSM_B200_ERROR_CLASS(SingularMatrix)
ASDSM_B200_ERROR_CLASS(SkeletonNotHollow)
ASDSM_B200_ERROR_CLASS(ZeroNormSolution)
ASDSM_B200_ERROR_CLASS(UnknownExample)
ASDSM_B200_ERROR_CLASS(NoExactSolution)
ASDSM_B200_ERROR_CLASS(Unsupported)  // outside the B200 path's scope (no reference class)
ASDSM_B200_ERROR_CLASS(CudaFailure)  // CUDA runtime failure: no GPU, out of memory, ...
#undef ASDSM_B200_ERROR_CLASS

inline void check(int rc) {
  if (rc == ASDSM_OK) return;
  const std::string msg = asdsm_last_error();
  switch (rc) {
    case ASDSM_DIVISIBILITY_ERROR: throw DivisibilityError(msg);
    case ASDSM_DEGENERATE_ERROR: throw DegenerateError(msg);
    case ASDSM_INDEX_OUT_OF_RANGE: throw IndexOutOfRange(msg);
    case ASDSM_NOT_A_SUBMESH: throw NotASubmesh(msg);
    case ASDSM_INVALID_KIND: throw InvalidKind(msg);
    case ASDSM_DIMENSION_MISMATCH: throw DimensionMismatch(msg);
    case ASDSM_SINGULAR_MATRIX: throw SingularMatrix(msg);
    case ASDSM_SKELETON_NOT_HOLLOW: throw SkeletonNotHollow(msg);
    case ASDSM_ZERO_NORM_SOLUTION: throw ZeroNormSolution(msg);
    case ASDSM_UNKNOWN_EXAMPLE: throw UnknownExample(msg);
    case ASDSM_NO_EXACT_SOLUTION: throw NoExactSolution(msg);
    case ASDSM_UNSUPPORTED: throw Unsupported(msg);
    case ASDSM_CUDA_FAILURE: throw CudaFailure(msg);
    default: throw Error(msg);
  }
}

// ---- mesh (mesh.hpp:22-83) --------------------------------------------------------------
// MeshKind as the coarse-axis bitmask of the C-ABI (bit a set: coarse along axis a).
struct MeshKind {
  unsigned mask = 0;
  bool holes = false;
  static MeshKind fine(int) { return {0u, false}; }
  static MeshKind coarse(int dim) { return {(1u << dim) - 1u, false}; }
  static MeshKind coarse_along(int, int axis) { return {1u << axis, false}; }
  static MeshKind holes_kind(int) { return {0u, true}; }
};

struct MeshConfig {
  int dim = 2;
  std::vector<int> fine_counts, coarse_counts, factors;
  int time_axis = -1;

  // MeshConfig::create (mesh.hpp:68, mesh.cpp:47-76): same validation and exceptions
  static MeshConfig create(int dim, std::vector<int> fine, std::vector<int> coarse, int time_axis = -1) {
    if (dim < 2 || dim > 3) throw DimensionMismatch("mesh dimension must be 2 or 3");
    if (static_cast<int>(fine.size()) != dim || static_cast<int>(coarse.size()) != dim)
      throw DimensionMismatch("mesh counts must have one entry per axis");
    if (time_axis != -1 && time_axis != dim - 1) throw DimensionMismatch("time axis must be the last axis");
    MeshConfig c;
    c.dim = dim;
    c.fine_counts = fine;
    c.coarse_counts = coarse;
    c.time_axis = time_axis;
    for (int a = 0; a < dim; ++a) {
      if (fine[a] < 1 || coarse[a] < 1) throw DegenerateError("interior point counts must be >= 1");
      if ((fine[a] + 1) % (coarse[a] + 1) != 0)
        throw DivisibilityError("fine intervals not divisible by coarse intervals on axis " + std::to_string(a));
      const int n = (fine[a] + 1) / (coarse[a] + 1);
      if (n < 2) throw DegenerateError("refinement factor 1 leaves no holes");
      c.factors.push_back(n);
    }
    return c;
  }

  // MeshConfig::point_count (mesh.hpp:72)
  std::int64_t point_count(const MeshKind& kind) const {
    std::int64_t n = 1;
    for (int a = 0; a < dim; ++a) {
      if (kind.holes) n *= static_cast<std::int64_t>(coarse_counts[a] + 1) * (factors[a] - 1);
      else n *= (kind.mask >> a & 1u) ? coarse_counts[a] : fine_counts[a];
    }
    return n;
  }
};

// ---- problems (problems.hpp:20-29) ------------------------------------------------------
class ProblemSpec {
 public:
  explicit ProblemSpec(asdsm_problem* h, std::shared_ptr<void> keep = nullptr)
      : h_(h, asdsm_problem_destroy), keep_(std::move(keep)) {
    double al[3], be[3];
    check(asdsm_problem_info(h, &dim_, &time_dependent_, &constant_coeffs_, al, be, &has_exact_));
  }
  asdsm_problem* handle() const { return h_.get(); }
  int dim() const { return dim_; }
  bool time_dependent() const { return time_dependent_ != 0; }
  bool constant_coefficients() const { return constant_coeffs_ != 0; }
  bool has_exact() const { return has_exact_ != 0; }

  // assemble_rhs (fdm.hpp:44-46) on a tensor kind
  std::vector<double> assemble_rhs(const MeshConfig& c, const MeshKind& kind) const {
    if (kind.holes) throw InvalidKind("holes have no standalone right-hand side");
    std::vector<double> out(static_cast<size_t>(c.point_count(kind)));
    check(asdsm_assemble_rhs(h_.get(), c.dim, c.fine_counts.data(), c.coarse_counts.data(), c.time_axis, kind.mask,
                             out.data()));
    return out;
  }
  std::vector<double> sample_exact(const MeshConfig& c) const {
    std::vector<double> out(static_cast<size_t>(c.point_count(MeshKind::fine(c.dim))));
    check(asdsm_sample_exact(h_.get(), c.dim, c.fine_counts.data(), c.coarse_counts.data(), c.time_axis, out.data()));
    return out;
  }

 private:
  std::shared_ptr<asdsm_problem> h_;
  std::shared_ptr<void> keep_;  // caller-defined fields the library calls back into
  int dim_ = 0, time_dependent_ = 0, constant_coeffs_ = 0, has_exact_ = 0;
};

// A caller-defined problem (fdm.hpp:17-30): the reference's ProblemSpec fields as callables of a
// point (axes beyond dim are zero), passed to the library as callbacks (asdsm_problem_create).
using Coord = std::array<double, 3>;
using ScalarField = std::function<double(const Coord&)>;
struct FieldSpec {
  int dim = 2;
  bool time_dependent = false;
  std::array<ScalarField, 3> alpha{}, beta{};  // per spatial axis
  ScalarField source, boundary, exact;         // exact optional
  int spatial_axes() const { return time_dependent ? dim - 1 : dim; }
};

inline ProblemSpec make_problem(const FieldSpec& fields) {
  auto keep = std::make_shared<FieldSpec>(fields);
  auto call = [](const double* x, void* ctx) {
    const Coord c{x[0], x[1], x[2]};
    return (*static_cast<const ScalarField*>(ctx))(c);
  };
  auto field = [&](const ScalarField& f) { return asdsm_field{f ? +call : nullptr, const_cast<ScalarField*>(&f)}; };
  asdsm_problem_spec spec{};
  spec.dim = keep->dim;
  spec.time_dependent = keep->time_dependent ? 1 : 0;
  for (int a = 0; a < keep->spatial_axes(); ++a) {
    spec.alpha[a] = field(keep->alpha[static_cast<size_t>(a)]);
    spec.beta[a] = field(keep->beta[static_cast<size_t>(a)]);
  }
  spec.source = field(keep->source);
  spec.boundary = field(keep->boundary);
  spec.exact = field(keep->exact);
  asdsm_problem* h = nullptr;
  check(asdsm_problem_create(&spec, &h));
  return ProblemSpec(h, keep);
}

inline ProblemSpec make_problem(int example, int setting) {  // problems.hpp:20
  asdsm_problem* h = nullptr;
  check(asdsm_problem_example(example, setting, &h));
  return ProblemSpec(h);
}

// The BASELINE.json configurations (seeded synthetic sources), with their meshes.
inline ProblemSpec baseline_problem(int config_id, std::uint64_t seed = 0) {
  asdsm_problem* h = nullptr;
  check(asdsm_problem_config(config_id, seed, &h));
  return ProblemSpec(h);
}
inline MeshConfig baseline_mesh(int config_id, int* iterations = nullptr) {
  int dim = 0, nf[3], nc[3], ta = -1, it = 0;
  check(asdsm_config_mesh(config_id, &dim, nf, nc, &ta, &it));
  if (iterations) *iterations = it;
  return MeshConfig::create(dim, std::vector<int>(nf, nf + dim), std::vector<int>(nc, nc + dim), ta);
}

inline MeshConfig example_mesh(int example, int setting, int nf, int nc) {  // problems.hpp:23
  const ProblemSpec p = make_problem(example, setting);
  return MeshConfig::create(p.dim(), std::vector<int>(p.dim(), nf), std::vector<int>(p.dim(), nc),
                            p.time_dependent() ? p.dim() - 1 : -1);
}

// ---- solver (solver.hpp:37-163) ---------------------------------------------------------
struct RhsBundle {  // solver.hpp:37-42
  std::vector<double> fine;
  std::vector<std::vector<double>> aniso;
  std::vector<double> coarse;
};

struct IterationRecord {  // solver.hpp:44-52
  int k = 0;
  double res_l2 = 0.0, res_inf = 0.0, err_max = 0.0, err_l2 = 0.0, s_hat = 0.0, wall_ms = 0.0;
};

struct IterationState {  // solver.hpp:54-59 (u, r: GridFunction::values on the fine kind)
  std::vector<double> u, r;
  std::vector<IterationRecord> history;
  std::string stop_reason;  // "tol" | "max_iter" | "stagnation"
};

struct IterateOptions {  // solver.hpp:56-68
  double tol = 1e-12;
  int max_iter = 20;
  int stagnation_window = 3;
  double stagnation_ratio = 0.99;
  double subsample = 0.0;
  std::uint64_t rng_seed = 0;
  bool sparse_residual = false;
  // called after each recorded iteration, k = 0 first (asdsm_iterate_observed: the solve runs
  // launch by launch with one synchronize per iteration instead of the captured graph)
  std::function<void(const IterationState&)> observer;
};

// SolverContext (solver.hpp:114-155): device-resident operators, tables and rhs bundle.
class SolverContext {
 public:
  SolverContext(const MeshConfig& config, const ProblemSpec& problem) : config_(config), problem_(problem) {
    if (problem.dim() != config.dim) throw DimensionMismatch("problem/mesh dimension mismatch");
    if (problem.time_dependent() != (config.time_axis >= 0))
      throw DimensionMismatch("problem and mesh disagree about a time axis");
    asdsm_plan* p = nullptr;
    check(asdsm_plan_create_problem(problem.handle(), config.dim, config.fine_counts.data(),
                                    config.coarse_counts.data(), config.time_axis, &p));
    plan_.reset(p, asdsm_plan_destroy);
    bundle_ = assembled_bundle();
    if (problem.has_exact()) exact_ = problem.sample_exact(config);
    set_bundle(bundle_);
  }

  const MeshConfig& config() const { return config_; }
  const ProblemSpec& problem() const { return problem_; }
  asdsm_plan* plan() const { return plan_.get(); }

  RhsBundle assembled_bundle() const {  // solver.hpp:125
    RhsBundle b;
    b.fine = problem_.assemble_rhs(config_, MeshKind::fine(config_.dim));
    for (int a = 0; a < config_.dim; ++a) b.aniso.push_back(problem_.assemble_rhs(config_, MeshKind::coarse_along(config_.dim, a)));
    b.coarse = problem_.assemble_rhs(config_, MeshKind::coarse(config_.dim));
    return b;
  }

  void set_bundle(const RhsBundle& b) {
    const double* slabs[3] = {nullptr, nullptr, nullptr};
    for (int a = 0; a < config_.dim; ++a) slabs[a] = b.aniso[static_cast<size_t>(a)].data();
    check(asdsm_set_bundle(plan_.get(), b.fine.data(), slabs, b.coarse.data(), exact_.empty() ? nullptr : exact_.data(), 0));
    bundle_ = b;
  }

  std::vector<double> residual(const std::vector<double>& u) const {  // fdm.hpp:50
    std::vector<double> r(u.size());
    check(asdsm_residual(plan_.get(), u.data(), bundle_.fine.data(), r.data()));
    return r;
  }
  std::vector<double> initial_guess() const {  // solver.hpp:132 (smooth mode, assembled bundle)
    std::vector<double> u(static_cast<size_t>(config_.point_count(MeshKind::fine(config_.dim))));
    check(asdsm_initial_guess(plan_.get(), u.data()));
    return u;
  }
  std::vector<double> error_guess(const std::vector<double>& r, std::uint64_t rng_seed) const {  // solver.hpp:135
    std::vector<double> e(r.size());
    check(asdsm_error_guess(plan_.get(), r.data(), rng_seed, e.data()));
    return e;
  }
  double optimal_scaling(const std::vector<double>& r, const std::vector<double>& e) const {  // solver.hpp:109
    double s = 0.0;
    check(asdsm_optimal_scaling(plan_.get(), r.data(), e.data(), &s));
    return s;
  }

  IterationState iterate(const IterateOptions& o) const { return run(o, nullptr); }

  // New right-hand sides and a solve in one call (C-ABI asdsm_solve: uploads, solve and
  // downloads ordered on the plan's stream, one synchronize).
  IterationState solve(const RhsBundle& b, const IterateOptions& o) {
    bundle_ = b;
    return run(o, &bundle_);
  }

 private:
  IterationState run(const IterateOptions& o, const RhsBundle* b) const {
    asdsm_iterate_options c{o.tol, o.max_iter, o.stagnation_window, o.stagnation_ratio, o.subsample, o.rng_seed,
                            o.sparse_residual ? 1 : 0};
    const size_t n = static_cast<size_t>(config_.point_count(MeshKind::fine(config_.dim)));
    IterationState st;
    st.u.resize(n);
    st.r.resize(n);
    std::vector<double> hist(7 * (static_cast<size_t>(std::max(o.max_iter, 0)) + 1));
    int nrec = 0, stop = 0;
    if (b) {
      const double* slabs[3] = {nullptr, nullptr, nullptr};
      for (int a = 0; a < config_.dim; ++a) slabs[a] = b->aniso[static_cast<size_t>(a)].data();
      check(asdsm_solve(plan_.get(), b->fine.data(), slabs, b->coarse.data(), exact_.empty() ? nullptr : exact_.data(),
                        &c, hist.data(), &nrec, &stop, st.u.data(), st.r.data()));
    } else if (o.observer) {
      auto obs = [](const double* h, int nr, const double* u, const double* r, std::int64_t nn, void* ctx) {
        IterationState s;
        s.u.assign(u, u + nn);
        s.r.assign(r, r + nn);
        for (int k = 0; k < nr; ++k)
          s.history.push_back({static_cast<int>(h[7 * k]), h[7 * k + 1], h[7 * k + 2], h[7 * k + 3], h[7 * k + 4],
                               h[7 * k + 5], h[7 * k + 6]});
        (*static_cast<const std::function<void(const IterationState&)>*>(ctx))(s);
      };
      check(asdsm_iterate_observed(plan_.get(), &c, obs, const_cast<std::function<void(const IterationState&)>*>(&o.observer),
                                   hist.data(), &nrec, &stop, st.u.data(), st.r.data()));
    } else {
      check(asdsm_iterate(plan_.get(), &c, hist.data(), &nrec, &stop, st.u.data(), st.r.data()));
    }
    for (int k = 0; k < nrec; ++k) {
      const double* h = hist.data() + 7 * k;
      st.history.push_back({static_cast<int>(h[0]), h[1], h[2], h[3], h[4], h[5], h[6]});
    }
    st.stop_reason = stop == ASDSM_STOP_TOL ? "tol" : stop == ASDSM_STOP_STAGNATION ? "stagnation" : "max_iter";
    return st;
  }

 private:
  MeshConfig config_;
  ProblemSpec problem_;
  std::shared_ptr<asdsm_plan> plan_;
  RhsBundle bundle_;
  std::vector<double> exact_;
};

// asdsm_iterate (solver.hpp:161-163)
inline IterationState asdsm_iterate(const ProblemSpec& problem, const MeshConfig& config,
                                    const IterateOptions& options = {}) {
  return SolverContext(config, problem).iterate(options);
}

}  // namespace asdsm_b200
