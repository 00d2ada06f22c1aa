// The reference-side binding (INTEGRATION.md "Reference-side binding"): the function a maintainer
// of the reference adds to proj/ so that callers keep the reference's own types.
// asdsm_iterate_b200 has asdsm_iterate's signature (solver.hpp:160-161) and runs the solve on the
// B200 through the C-ABI (include/asdsm_b200.h): the caller's ProblemSpec fields (fdm.hpp:17-30)
// go in as callbacks, the right-hand sides are assembled exactly as SolverContext does, the
// IterateOptions (observer included) map onto asdsm_iterate / asdsm_iterate_observed, and the
// C-ABI status codes come back as the errors.hpp exception classes.
//
// Test driver (tests/test_gpu_binding.py; built by oracle/Makefile against the reference's
// headers and library):
//   ref_binding CASE NF NC ITERS SEED PREFIX
// CASE: ex:E:S (make_problem(E, S) on example_mesh) | adv:EPS (a caller-defined advection-
// dominated problem: alpha = EPS, beta = (1, 0.5), two source bumps, g = 0) | var (a
// caller-defined variable-coefficient problem outside the reference's catalogue).
// Runs the reference's own asdsm_iterate and asdsm_iterate_b200 on the same ProblemSpec and
// writes PREFIX.{ref,gpu}.hist.txt (k res_l2 res_inf err_max err_l2 s_hat per row) and
// PREFIX.{ref,gpu}.u.f64; PREFIX.obs.txt holds the observer's (k, res_l2) calls.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <memory>
#include <string>
#include <vector>

#include "asdsm/errors.hpp"
#include "asdsm/problems.hpp"
#include "asdsm/solver.hpp"
#include "asdsm_b200.h"

namespace asdsm_b200_binding {

double field_call(const double* x, void* ctx) {
  const auto& f = *static_cast<const asdsm::ScalarField*>(ctx);
  asdsm::Coord c{};
  for (int a = 0; a < asdsm::kMaxDim; ++a) c[static_cast<std::size_t>(a)] = x[a];
  return f(c);
}

[[noreturn]] void raise(int rc) {
  const std::string msg = asdsm_last_error();
  switch (rc) {
    case ASDSM_DIVISIBILITY_ERROR: throw asdsm::DivisibilityError(msg);
    case ASDSM_DEGENERATE_ERROR: throw asdsm::DegenerateError(msg);
    case ASDSM_INDEX_OUT_OF_RANGE: throw asdsm::IndexOutOfRange(msg);
    case ASDSM_NOT_A_SUBMESH: throw asdsm::NotASubmesh(msg);
    case ASDSM_INVALID_KIND: throw asdsm::InvalidKind(msg);
    case ASDSM_DIMENSION_MISMATCH: throw asdsm::DimensionMismatch(msg);
    case ASDSM_SINGULAR_MATRIX: throw asdsm::SingularMatrix(msg);
    case ASDSM_SKELETON_NOT_HOLLOW: throw asdsm::SkeletonNotHollow(msg);
    case ASDSM_ZERO_NORM_SOLUTION: throw asdsm::ZeroNormSolution(msg);
    case ASDSM_UNKNOWN_EXAMPLE: throw asdsm::UnknownExample(msg);
    case ASDSM_NO_EXACT_SOLUTION: throw asdsm::NoExactSolution(msg);
    default: throw asdsm::Error(msg);
  }
}

void check(int rc) {
  if (rc != ASDSM_OK) raise(rc);
}

asdsm::IterationRecord record(const double* row) {
  return {static_cast<int>(row[0]), row[1], row[2], row[3], row[4], row[5], row[6]};
}

struct ObserverCtx {
  const asdsm::IterateOptions* options;
  asdsm::MeshKind kind;
};

void observe(const double* history, int nrec, const double* u, const double* r, int64_t n, void* ctx) {
  const auto* oc = static_cast<const ObserverCtx*>(ctx);
  asdsm::IterationState st;
  st.u = asdsm::GridFunction(oc->kind, std::vector<double>(u, u + n));
  st.r = asdsm::GridFunction(oc->kind, std::vector<double>(r, r + n));
  for (int k = 0; k < nrec; ++k) st.history.push_back(record(history + 7 * k));
  oc->options->observer(st);
}

asdsm::IterationState asdsm_iterate_b200(const asdsm::ProblemSpec& p, const asdsm::MeshConfig& c,
                                         const asdsm::IterateOptions& o = {}) {
  asdsm_problem_spec spec{};
  spec.dim = p.dim;
  spec.time_dependent = p.time_dependent ? 1 : 0;
  auto field = [](const asdsm::ScalarField& f) {
    return asdsm_field{field_call, const_cast<asdsm::ScalarField*>(&f)};
  };
  for (int a = 0; a < p.spatial_axes(); ++a) {
    spec.alpha[a] = field(p.alpha[static_cast<std::size_t>(a)]);
    spec.beta[a] = field(p.beta[static_cast<std::size_t>(a)]);
  }
  spec.source = field(p.source);
  spec.boundary = field(p.boundary);
  if (p.exact) spec.exact = field(p.exact);
  asdsm_problem* prob = nullptr;
  check(asdsm_problem_create(&spec, &prob));
  std::unique_ptr<asdsm_problem, void (*)(asdsm_problem*)> hold_prob(prob, asdsm_problem_destroy);
  const int* fc = c.fine_counts.data();
  const int* cc = c.coarse_counts.data();
  asdsm_plan* plan = nullptr;
  check(asdsm_plan_create_problem(prob, c.dim, fc, cc, c.time_axis, &plan));
  std::unique_ptr<asdsm_plan, void (*)(asdsm_plan*)> hold_plan(plan, asdsm_plan_destroy);

  // the right-hand sides SolverContext::assembled_bundle holds (solver.hpp:127, fdm.hpp:44)
  const asdsm::MeshKind fine_kind = asdsm::MeshKind::fine(c.dim);
  const auto nf = c.point_count(fine_kind);
  std::vector<double> fine(static_cast<std::size_t>(nf));
  std::vector<double> coarse(static_cast<std::size_t>(c.point_count(asdsm::MeshKind::coarse(c.dim))));
  std::vector<std::vector<double>> slab(static_cast<std::size_t>(c.dim));
  check(asdsm_assemble_rhs(prob, c.dim, fc, cc, c.time_axis, 0u, fine.data()));
  const double* slabs[3] = {nullptr, nullptr, nullptr};
  for (int a = 0; a < c.dim; ++a) {
    auto& s = slab[static_cast<std::size_t>(a)];
    s.resize(static_cast<std::size_t>(c.point_count(asdsm::MeshKind::coarse_along(c.dim, a))));
    check(asdsm_assemble_rhs(prob, c.dim, fc, cc, c.time_axis, 1u << a, s.data()));
    slabs[a] = s.data();
  }
  check(asdsm_assemble_rhs(prob, c.dim, fc, cc, c.time_axis, (1u << c.dim) - 1u, coarse.data()));
  std::vector<double> exact;
  if (p.exact) {
    exact.resize(static_cast<std::size_t>(nf));
    check(asdsm_sample_exact(prob, c.dim, fc, cc, c.time_axis, exact.data()));
  }
  check(asdsm_set_bundle(plan, fine.data(), slabs, coarse.data(), exact.empty() ? nullptr : exact.data(), 0));

  const asdsm_iterate_options opt{o.tol,         o.max_iter,   o.stagnation_window,
                                  o.stagnation_ratio, o.subsample, o.rng_seed,
                                  o.sparse_residual ? 1 : 0};
  asdsm::IterationState st;
  st.u = asdsm::GridFunction(fine_kind, nf);
  st.r = asdsm::GridFunction(fine_kind, nf);
  std::vector<double> hist(static_cast<std::size_t>(7 * (std::max(o.max_iter, 0) + 1)));
  int nrec = 0, stop = 0;
  if (o.observer) {
    ObserverCtx ctx{&o, fine_kind};
    check(asdsm_iterate_observed(plan, &opt, observe, &ctx, hist.data(), &nrec, &stop, st.u.values.data(),
                                 st.r.values.data()));
  } else {
    check(asdsm_iterate(plan, &opt, hist.data(), &nrec, &stop, st.u.values.data(), st.r.values.data()));
  }
  for (int k = 0; k < nrec; ++k) st.history.push_back(record(hist.data() + 7 * k));
  st.stop_reason = stop == ASDSM_STOP_TOL ? "tol" : stop == ASDSM_STOP_STAGNATION ? "stagnation" : "max_iter";
  return st;
}

}  // namespace asdsm_b200_binding

namespace {

double bump(double x, double y, double cx, double cy, double w) {
  const double dx = x - cx, dy = y - cy;
  return std::exp(-(dx * dx + dy * dy) / (2.0 * w * w));
}

void write_state(const std::string& prefix, const asdsm::IterationState& st) {
  std::ofstream h(prefix + ".hist.txt");
  char line[256];
  for (const auto& r : st.history) {
    std::snprintf(line, sizeof line, "%d %.17g %.17g %.17g %.17g %.17g\n", r.k, r.res_l2, r.res_inf, r.err_max,
                  r.err_l2, r.s_hat);
    h << line;
  }
  h << "# stop: " << st.stop_reason << "\n";
  std::ofstream u(prefix + ".u.f64", std::ios::binary);
  u.write(reinterpret_cast<const char*>(st.u.values.data()),
          static_cast<std::streamsize>(st.u.values.size() * sizeof(double)));
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 7) {
    std::fprintf(stderr, "usage: ref_binding CASE NF NC ITERS SEED PREFIX\n");
    return 2;
  }
  const std::string which = argv[1];
  const int nf = std::atoi(argv[2]), nc = std::atoi(argv[3]), iters = std::atoi(argv[4]);
  const std::uint64_t seed = std::strtoull(argv[5], nullptr, 10);
  const std::string prefix = argv[6];
  asdsm::ProblemSpec problem;
  asdsm::MeshConfig mesh;
  if (which.rfind("ex:", 0) == 0) {
    int e = 0, s = 0;
    std::sscanf(which.c_str(), "ex:%d:%d", &e, &s);
    problem = asdsm::make_problem(e, s);
    mesh = asdsm::example_mesh(e, s, nf, nc);
  } else if (which.rfind("adv:", 0) == 0) {
    const double eps = std::atof(which.c_str() + 4);
    problem.dim = 2;
    problem.alpha = {[eps](const asdsm::Coord&) { return eps; }, [eps](const asdsm::Coord&) { return eps; }, {}};
    problem.beta = {[](const asdsm::Coord&) { return 1.0; }, [](const asdsm::Coord&) { return 0.5; }, {}};
    problem.source = [](const asdsm::Coord& x) {
      return bump(x[0], x[1], 0.3, 0.4, 0.1) - 0.5 * bump(x[0], x[1], 0.7, 0.6, 0.15);
    };
    problem.boundary = [](const asdsm::Coord&) { return 0.0; };
    const int n[2] = {nf, nf}, m[2] = {nc, nc};
    mesh = asdsm::MeshConfig::create(2, n, m);
  } else if (which == "var") {
    problem.dim = 2;
    problem.alpha = {[](const asdsm::Coord& x) { return 0.5 + x[1] * x[1]; },
                     [](const asdsm::Coord& x) { return 1.0 + 0.5 * std::sin(3.0 * x[0]); }, {}};
    problem.beta = {[](const asdsm::Coord& x) { return 1.0 - x[1]; }, [](const asdsm::Coord& x) { return x[0]; }, {}};
    problem.exact = [](const asdsm::Coord& x) { return x[0] * (1.0 - x[0]) * std::sin(2.0 * x[1]); };
    problem.source = [](const asdsm::Coord& x) { return 1.0 + x[0] * x[1]; };
    problem.boundary = problem.exact;
    const int n[2] = {nf, nf}, m[2] = {nc, nc};
    mesh = asdsm::MeshConfig::create(2, n, m);
  } else {
    std::fprintf(stderr, "unknown case %s\n", which.c_str());
    return 2;
  }
  asdsm::IterateOptions opts;
  opts.tol = 0.0;
  opts.max_iter = iters;
  opts.stagnation_window = 0;
  opts.rng_seed = seed;
  try {
    const asdsm::IterationState ref = asdsm::asdsm_iterate(problem, mesh, opts);
    write_state(prefix + ".ref", ref);
    std::ofstream obs(prefix + ".obs.txt");
    opts.observer = [&obs](const asdsm::IterationState& st) {
      char line[96];
      std::snprintf(line, sizeof line, "%d %.17g\n", st.history.back().k, st.history.back().res_l2);
      obs << line;
    };
    const asdsm::IterationState gpu = asdsm_b200_binding::asdsm_iterate_b200(problem, mesh, opts);
    write_state(prefix + ".gpu", gpu);
  } catch (const asdsm::Error& e) {
    std::fprintf(stderr, "asdsm error: %s\n", e.what());
    return 3;
  }
  return 0;
}
