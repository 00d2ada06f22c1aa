// C-ABI layer (include/asdsm_b200.h) over the B200 Solver.  Thin: argument validation,
// error-code translation, host<->device copies for the host-pointer entry points.
#include "../../include/asdsm_b200.h"

#include <cstring>
#include <functional>
#include <memory>
#include <string>
#include <vector>

#include "../../include/asdsm_problems.hpp"
#include "assemble.hpp"
#include "solver.hpp"

using namespace asdsm_b200;

struct asdsm_plan {
  std::unique_ptr<Solver> solver;
  cudaStream_t stream = nullptr;
  int max_iter_run = 0;
};

struct asdsm_problem {
  asdsm_cat::Problem p;
  bool callbacks = false;  // caller-defined fields: constant or variable decided per plan
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return ASDSM_OK;
  } catch (const AsdsmError& e) {
    g_last_error = e.what();
    return e.code;
  } catch (const CudaError& e) {
    g_last_error = e.what();
    return ASDSM_CUDA_FAILURE;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return ASDSM_UNKNOWN_EXAMPLE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return ASDSM_ERROR;
  }
}

Mesh mesh_from(int dim, const int* nf, const int* nc, int time_axis) { return Mesh::create(dim, nf, nc, time_axis); }

cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

}  // namespace

extern "C" {

const char* asdsm_last_error(void) { return g_last_error.c_str(); }
int asdsm_abi_version(void) { return ASDSM_B200_ABI_VERSION; }

void asdsm_default_options(asdsm_iterate_options* o) {
  o->tol = 1e-12;
  o->max_iter = 20;
  o->stagnation_window = 3;
  o->stagnation_ratio = 0.99;
  o->subsample = 0.0;
  o->rng_seed = 0;
  o->sparse_residual = 0;
}

int asdsm_problem_example(int example, int setting, asdsm_problem** out) {
  return guarded([&] {
    if (example < 1 || example > 4 || (setting != 1 && setting != 2))
      throw AsdsmError(kUnknownExample, "example must be 1..4 and setting 1 or 2");
    auto* p = new asdsm_problem;
    p->p = asdsm_cat::reference_example(example, setting);
    *out = p;
  });
}

int asdsm_problem_config(int config_id, uint64_t seed, asdsm_problem** out) {
  return guarded([&] {
    if (config_id < 0 || config_id >= asdsm_cat::kNumBaselineConfigs)
      throw AsdsmError(kUnknownExample, "config id must be 0..4");
    auto* p = new asdsm_problem;
    p->p = asdsm_cat::baseline_problem(config_id, seed);
    *out = p;
  });
}

int asdsm_problem_create(const asdsm_problem_spec* spec, asdsm_problem** out) {
  return guarded([&] {
    if (!spec || !out) throw AsdsmError(kError, "null problem spec");
    if (spec->dim != 2 && spec->dim != 3) throw AsdsmError(kDimensionMismatch, "problem dimension must be 2 or 3");
    const int ns = spec->dim - (spec->time_dependent ? 1 : 0);
    auto wrap = [&](const asdsm_field& f, const char* what) -> asdsm_cat::Field {
      if (!f.fn) throw AsdsmError(kError, std::string("problem field missing: ") + what);
      const asdsm_field_fn fn = f.fn;
      void* ctx = f.ctx;
      return [fn, ctx](const asdsm_cat::Coord& x) { return fn(x.data(), ctx); };
    };
    auto p = std::make_unique<asdsm_problem>();
    p->callbacks = true;
    p->p.dim = spec->dim;
    p->p.time_dependent = spec->time_dependent != 0;
    for (int a = 0; a < ns; ++a) {
      p->p.alpha[static_cast<size_t>(a)] = wrap(spec->alpha[a], "alpha");
      p->p.beta[static_cast<size_t>(a)] = wrap(spec->beta[a], "beta");
    }
    p->p.source = wrap(spec->source, "source");
    p->p.boundary = wrap(spec->boundary, "boundary");
    if (spec->exact.fn) p->p.exact = wrap(spec->exact, "exact");
    p->p.constant_coeffs = false;
    *out = p.release();
  });
}

void asdsm_problem_destroy(asdsm_problem* p) { delete p; }

int asdsm_problem_info(const asdsm_problem* p, int* dim, int* time_dependent, int* constant_coeffs, double* alpha,
                       double* beta, int* has_exact) {
  return guarded([&] {
    *dim = p->p.dim;
    *time_dependent = p->p.time_dependent;
    *constant_coeffs = p->p.constant_coeffs;
    for (int a = 0; a < 3; ++a) {
      alpha[a] = p->p.alpha_c[static_cast<size_t>(a)];
      beta[a] = p->p.beta_c[static_cast<size_t>(a)];
    }
    *has_exact = static_cast<bool>(p->p.exact);
  });
}

int asdsm_config_mesh(int config_id, int* dim, int* fine_counts, int* coarse_counts, int* time_axis, int* iterations) {
  return guarded([&] {
    if (config_id < 0 || config_id >= asdsm_cat::kNumBaselineConfigs)
      throw AsdsmError(kUnknownExample, "config id must be 0..4");
    const auto m = asdsm_cat::baseline_mesh(config_id);
    *dim = m.dim;
    for (int a = 0; a < 3; ++a) {
      fine_counts[a] = m.nf[static_cast<size_t>(a)];
      coarse_counts[a] = m.nc[static_cast<size_t>(a)];
    }
    *time_axis = m.time_axis;
    *iterations = m.iterations;
  });
}

int asdsm_assemble_rhs(const asdsm_problem* p, int dim, const int* fine_counts, const int* coarse_counts, int time_axis,
                       unsigned mask, double* out) {
  return guarded([&] {
    const Mesh m = mesh_from(dim, fine_counts, coarse_counts, time_axis);
    if (p->p.dim != dim) throw AsdsmError(kDimensionMismatch, "problem/mesh dimension mismatch");
    if (p->p.time_dependent != (time_axis >= 0))
      throw AsdsmError(kDimensionMismatch, "problem and mesh disagree about a time axis");
    if (mask >= (1u << dim)) throw AsdsmError(kIndexOutOfRange, "mask out of range");
    assemble_rhs(m, mask, p->p, out);
  });
}

int asdsm_sample_exact(const asdsm_problem* p, int dim, const int* fine_counts, const int* coarse_counts, int time_axis,
                       double* out) {
  return guarded([&] {
    if (!p->p.exact) throw AsdsmError(kNoExactSolution, "problem has no exact solution attached");
    const Mesh m = mesh_from(dim, fine_counts, coarse_counts, time_axis);
    sample_exact(m, p->p, out);
  });
}

int asdsm_plan_create(int dim, const int* fine_counts, const int* coarse_counts, int time_axis, const double* alpha,
                      const double* beta, asdsm_plan** out) {
  return guarded([&] {
    const Mesh m = mesh_from(dim, fine_counts, coarse_counts, time_axis);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw CudaError("no CUDA device: the B200 path has no CPU fallback");
    auto plan = std::make_unique<asdsm_plan>();
    ASDSM_CUDA_CHECK(cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking));
    plan->solver = std::make_unique<Solver>(m, alpha, beta);
    *out = plan.release();
  });
}

int asdsm_plan_create_problem(const asdsm_problem* problem, int dim, const int* fine_counts, const int* coarse_counts,
                              int time_axis, asdsm_plan** out) {
  return guarded([&] {
    const Mesh m = mesh_from(dim, fine_counts, coarse_counts, time_axis);
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
      throw CudaError("no CUDA device: the B200 path has no CPU fallback");
    auto plan = std::make_unique<asdsm_plan>();
    ASDSM_CUDA_CHECK(cudaStreamCreateWithFlags(&plan->stream, cudaStreamNonBlocking));
    if (problem->callbacks) {
      // caller-defined fields: constant coefficients iff every fine-node sample agrees (the
      // operator the reference assembles is then exactly the constant-coefficient one)
      asdsm_cat::Problem q = problem->p;
      if (q.dim != dim) throw AsdsmError(kDimensionMismatch, "problem/mesh dimension mismatch");
      q.constant_coeffs = uniform_coefficients(m, q, q.alpha_c.data(), q.beta_c.data());
      plan->solver = std::make_unique<Solver>(m, q);
    } else {
      plan->solver = std::make_unique<Solver>(m, problem->p);
    }
    *out = plan.release();
  });
}

int asdsm_plan_is_variable(const asdsm_plan* plan) { return plan->solver->variable() ? 1 : 0; }

void asdsm_plan_destroy(asdsm_plan* plan) {
  if (!plan) return;
  if (plan->stream) cudaStreamSynchronize(plan->stream);
  plan->solver.reset();
  if (plan->stream) cudaStreamDestroy(plan->stream);
  delete plan;
}

int asdsm_point_count(const asdsm_plan* plan, unsigned coarse_mask, int holes, int64_t* out) {
  return guarded([&] {
    const Mesh& m = plan->solver->mesh();
    if (holes) {
      *out = m.hole_count();
      return;
    }
    if (coarse_mask >= (1u << m.dim)) throw AsdsmError(kIndexOutOfRange, "from_mask: mask out of range");
    *out = m.point_count(coarse_mask);
  });
}

int asdsm_projector_map(asdsm_plan* plan, unsigned from_mask, unsigned to_mask, int to_holes, int64_t* out) {
  return guarded([&] {
    const Mesh& m = plan->solver->mesh();
    const unsigned full = (1u << m.dim) - 1u;
    if (from_mask > full || (!to_holes && to_mask > full)) throw AsdsmError(kIndexOutOfRange, "mask out of range");
    i64 count = 0;
    if (to_holes) {
      if (from_mask != 0) throw AsdsmError(kNotASubmesh, "holes are a subset of the fine mesh only");
      count = m.hole_count();
    } else {
      if ((from_mask & to_mask) != from_mask) throw AsdsmError(kNotASubmesh, "target is not a sub-mesh of the source");
      count = m.point_count(to_mask);
    }
    long long* d = nullptr;
    ASDSM_CUDA_CHECK(cudaMalloc(&d, static_cast<size_t>(count) * sizeof(long long) + 8));
    if (to_holes)
      launch_hole_map(plan->solver->mesh_dev(), d, count, plan->stream);
    else
      launch_projector_map(plan->solver->mesh_dev(), from_mask, to_mask, d, count, plan->stream);
    cudaError_t e = cudaMemcpyAsync(out, d, static_cast<size_t>(count) * sizeof(long long), cudaMemcpyDeviceToHost,
                                    plan->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(plan->stream);
    cudaFree(d);
    if (e != cudaSuccess) throw CudaError(cudaGetErrorString(e));
  });
}

int asdsm_set_bundle(asdsm_plan* plan, const double* b_fine, const double* const* b_slab, const double* b_coarse,
                     const double* exact, int on_device) {
  return guarded([&] {
    // synchronous in both cases: host buffers are free again, and device copies are complete
    // before any later call on any stream reads the bundle (the caller's producer of device
    // sources must have finished: synchronize it, or use asdsm_set_bundle_async on that stream)
    plan->solver->set_bundle(b_fine, b_slab, b_coarse, exact, on_device != 0, plan->stream);
    ASDSM_CUDA_CHECK(cudaStreamSynchronize(plan->stream));
  });
}

int asdsm_set_bundle_async(asdsm_plan* plan, const double* b_fine, const double* const* b_slab,
                           const double* b_coarse, const double* exact, int on_device, void* stream) {
  return guarded([&] {
    // stream-ordered: after the caller's producer work on `stream`, before its next
    // asdsm_iterate_async on `stream`
    plan->solver->set_bundle(b_fine, b_slab, b_coarse, exact, on_device != 0,
                             stream ? as_stream(stream) : plan->stream);
  });
}

static RunOptions to_run(const asdsm_iterate_options* o) {
  RunOptions r;
  if (o) {
    r.tol = o->tol;
    r.max_iter = o->max_iter;
    r.stagnation_window = o->stagnation_window;
    r.stagnation_ratio = o->stagnation_ratio;
    r.subsample = o->subsample;
    r.rng_seed = o->rng_seed;
  }
  if (o) r.sparse_residual = o->sparse_residual != 0;
  if (r.subsample < 0.0) r.subsample = 0.0;
  if (r.max_iter < 0) r.max_iter = 0;
  return r;
}

int asdsm_iterate_async(asdsm_plan* plan, const asdsm_iterate_options* opts, void* stream) {
  return guarded([&] {
    const RunOptions r = to_run(opts);
    plan->max_iter_run = r.max_iter;
    plan->solver->run(r, stream ? as_stream(stream) : plan->stream);
  });
}

int asdsm_fetch(asdsm_plan* plan, void* stream, double* history, int* nrec, int* stop_code, double* u_out, double* r_out) {
  return guarded([&] {
    cudaStream_t s = stream ? as_stream(stream) : plan->stream;
    std::vector<double> rows;
    int stop = 0;
    const int n = plan->solver->fetch(rows, stop, u_out, r_out, s);
    if (history && n > 0) std::memcpy(history, rows.data(), rows.size() * sizeof(double));
    if (nrec) *nrec = n;
    if (stop_code) *stop_code = stop;
  });
}

int asdsm_iterate(asdsm_plan* plan, const asdsm_iterate_options* opts, double* history, int* nrec, int* stop_code,
                  double* u_out, double* r_out) {
  const int rc = asdsm_iterate_async(plan, opts, nullptr);
  if (rc != ASDSM_OK) return rc;
  return asdsm_fetch(plan, nullptr, history, nrec, stop_code, u_out, r_out);
}

int asdsm_iterate_observed(asdsm_plan* plan, const asdsm_iterate_options* opts, asdsm_observer_fn observer,
                           void* ctx, double* history, int* nrec, int* stop_code, double* u_out, double* r_out) {
  const int rc = guarded([&] {
    const RunOptions r = to_run(opts);
    plan->max_iter_run = r.max_iter;
    Solver& S = *plan->solver;
    const size_t n = static_cast<size_t>(S.fine_size());
    std::vector<double> rows, u(observer ? n : 0), res(observer ? n : 0);
    std::function<bool(int)> hook = [&](int) {
      bool active = true;
      const int nr = S.snapshot(rows, active, observer ? u.data() : nullptr, observer ? res.data() : nullptr,
                                plan->stream);
      if (observer) observer(rows.data(), nr, u.data(), res.data(), static_cast<int64_t>(n), ctx);
      return active;
    };
    S.run_observed(r, plan->stream, hook);
  });
  if (rc != ASDSM_OK) return rc;
  return asdsm_fetch(plan, nullptr, history, nrec, stop_code, u_out, r_out);
}

int asdsm_solve(asdsm_plan* plan, const double* b_fine, const double* const* b_slab, const double* b_coarse,
                const double* exact, const asdsm_iterate_options* opts, double* history, int* nrec, int* stop_code,
                double* u_out, double* r_out) {
  const int rc = guarded([&] {
    // stream-ordered uploads: the synchronize at the end of the fetch covers the host buffers
    plan->solver->set_bundle(b_fine, b_slab, b_coarse, exact, false, plan->stream);
  });
  if (rc != ASDSM_OK) return rc;
  return asdsm_iterate(plan, opts, history, nrec, stop_code, u_out, r_out);
}

int asdsm_device_solution(asdsm_plan* plan, void* stream, const double** u_dev) {
  return guarded([&] { *u_dev = plan->solver->u_current(stream ? as_stream(stream) : plan->stream); });
}

int64_t asdsm_last_launch_count(const asdsm_plan* plan) { return plan->solver->last_launches(); }

int asdsm_plan_kernels(const asdsm_plan* plan, char* buf, int64_t len) {
  return guarded([&] {
    std::string s;
    for (const auto& k : plan->solver->graph_kernels()) s += k.first + "\t" + std::to_string(k.second) + "\n";
    if (buf && len > 0) {
      const size_t n = std::min<size_t>(s.size(), static_cast<size_t>(len - 1));
      std::memcpy(buf, s.data(), n);
      buf[n] = 0;
    }
  });
}

void* asdsm_plan_stream(asdsm_plan* plan) { return plan->stream; }

int asdsm_profile_components(asdsm_plan* plan, void* stream, int reps, int max_components, char* names, double* ms,
                             double* bytes, double* flops, int* per_solve, int* count) {
  return guarded([&] {
    const auto comps = plan->solver->profile(stream ? as_stream(stream) : plan->stream, reps);
    const int n = std::min<int>(max_components, static_cast<int>(comps.size()));
    for (int i = 0; i < n; ++i) {
      std::strncpy(names + 64 * i, comps[static_cast<size_t>(i)].name.c_str(), 63);
      names[64 * i + 63] = 0;
      ms[i] = comps[static_cast<size_t>(i)].ms;
      bytes[i] = comps[static_cast<size_t>(i)].bytes;
      flops[i] = comps[static_cast<size_t>(i)].flops;
      per_solve[i] = comps[static_cast<size_t>(i)].per_solve;
    }
    *count = n;
  });
}

int asdsm_residual(asdsm_plan* plan, const double* u, const double* b, double* r) {
  return guarded([&] {
    Solver& S = *plan->solver;
    const size_t bytes = static_cast<size_t>(S.fine_size()) * sizeof(double);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.u_buffer(0), u, bytes, cudaMemcpyHostToDevice, plan->stream));
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.e_buffer(), b, bytes, cudaMemcpyHostToDevice, plan->stream));
    S.residual(S.u_buffer(0), S.e_buffer(), S.r_buffer(0), plan->stream);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(r, S.r_buffer(0), bytes, cudaMemcpyDeviceToHost, plan->stream));
    ASDSM_CUDA_CHECK(cudaStreamSynchronize(plan->stream));
  });
}

int asdsm_initial_guess(asdsm_plan* plan, double* u_out) {
  return guarded([&] {
    Solver& S = *plan->solver;
    const size_t bytes = static_cast<size_t>(S.fine_size()) * sizeof(double);
    S.initial_guess(S.u_buffer(0), 0, plan->stream);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(u_out, S.u_buffer(0), bytes, cudaMemcpyDeviceToHost, plan->stream));
    ASDSM_CUDA_CHECK(cudaStreamSynchronize(plan->stream));
  });
}

int asdsm_error_guess(asdsm_plan* plan, const double* r, uint64_t seed, double* e_out) {
  return guarded([&] {
    Solver& S = *plan->solver;
    const size_t bytes = static_cast<size_t>(S.fine_size()) * sizeof(double);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.r_buffer(0), r, bytes, cudaMemcpyHostToDevice, plan->stream));
    S.error_guess(S.r_buffer(0), seed, S.e_buffer(), plan->stream);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(e_out, S.e_buffer(), bytes, cudaMemcpyDeviceToHost, plan->stream));
    ASDSM_CUDA_CHECK(cudaStreamSynchronize(plan->stream));
  });
}

int asdsm_optimal_scaling(asdsm_plan* plan, const double* r, const double* e, double* s_out) {
  return guarded([&] {
    Solver& S = *plan->solver;
    const size_t bytes = static_cast<size_t>(S.fine_size()) * sizeof(double);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.r_buffer(0), r, bytes, cudaMemcpyHostToDevice, plan->stream));
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.e_buffer(), e, bytes, cudaMemcpyHostToDevice, plan->stream));
    *s_out = S.optimal_scaling(S.r_buffer(0), S.e_buffer(), plan->stream);
  });
}

// ---- public solver stages (solver.hpp:70-105) -------------------------------------------

int asdsm_richardson_extrapolate(asdsm_plan* plan, const double* u1_cc, const double* u2_cc, const double* u_cc,
                                 double* out) {
  return guarded([&] {
    Solver& S = *plan->solver;
    const size_t nb = static_cast<size_t>(S.kind_size((1u << S.mesh().dim) - 1u)) * sizeof(double);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.coarse_buffer(1), u1_cc, nb, cudaMemcpyHostToDevice, plan->stream));
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.coarse_buffer(2), u2_cc, nb, cudaMemcpyHostToDevice, plan->stream));
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.coarse_buffer(0), u_cc, nb, cudaMemcpyHostToDevice, plan->stream));
    S.stage_richardson(S.coarse_buffer(1), S.coarse_buffer(2), S.coarse_buffer(0), S.coarse_buffer(1), plan->stream);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(out, S.coarse_buffer(1), nb, cudaMemcpyDeviceToHost, plan->stream));
    ASDSM_CUDA_CHECK(cudaStreamSynchronize(plan->stream));
  });
}

int asdsm_choose_cross_points(asdsm_plan* plan, const double* u_fc, const double* u_cf, uint64_t rng_seed,
                              double* out) {
  return guarded([&] {
    Solver& S = *plan->solver;
    if (S.mesh().dim != 2) throw AsdsmError(kInvalidKind, "choose_cross_points: the 2D anisotropic meshes");
    const int axis = S.cross_point_choice(rng_seed) == 0 ? 0 : 1;  // u_cf is coarse along 0, u_fc along 1
    const size_t ns = static_cast<size_t>(S.kind_size(1u << axis)) * sizeof(double);
    const size_t nb = static_cast<size_t>(S.kind_size(3u)) * sizeof(double);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.slab_buffer(axis), axis == 0 ? u_cf : u_fc, ns, cudaMemcpyHostToDevice,
                                     plan->stream));
    S.stage_restrict(S.slab_buffer(axis), axis, S.coarse_buffer(1), plan->stream);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(out, S.coarse_buffer(1), nb, cudaMemcpyDeviceToHost, plan->stream));
    ASDSM_CUDA_CHECK(cudaStreamSynchronize(plan->stream));
  });
}

int asdsm_spline_correct(asdsm_plan* plan, const double* u_aniso, const double* e_cc, int dense_axis, double* out) {
  return guarded([&] {
    Solver& S = *plan->solver;
    if (S.mesh().dim != 2) throw AsdsmError(kInvalidKind, "spline correction applies to the 2D anisotropic meshes");
    if (dense_axis < 0 || dense_axis > 1) throw AsdsmError(kIndexOutOfRange, "dense_axis must be 0 or 1");
    const int other = 1 - dense_axis;
    const size_t ns = static_cast<size_t>(S.kind_size(1u << other)) * sizeof(double);
    const size_t nb = static_cast<size_t>(S.kind_size(3u)) * sizeof(double);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.slab_buffer(other), u_aniso, ns, cudaMemcpyHostToDevice, plan->stream));
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.coarse_buffer(1), e_cc, nb, cudaMemcpyHostToDevice, plan->stream));
    S.stage_spline_correct(S.slab_buffer(other), S.coarse_buffer(1), dense_axis, S.slab_buffer(other), plan->stream);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(out, S.slab_buffer(other), ns, cudaMemcpyDeviceToHost, plan->stream));
    ASDSM_CUDA_CHECK(cudaStreamSynchronize(plan->stream));
  });
}

namespace {
void skeleton_call(asdsm_plan* plan, const double* const* sol, const double* u_cc, uint64_t seed, double* out) {
  Solver& S = *plan->solver;
  const int dim = S.mesh().dim;
  double* dsol[3] = {nullptr, nullptr, nullptr};
  for (int a = 0; a < dim; ++a) {
    dsol[a] = S.slab_buffer(a);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(dsol[a], sol[a], static_cast<size_t>(S.kind_size(1u << a)) * sizeof(double),
                                     cudaMemcpyHostToDevice, plan->stream));
  }
  if (u_cc)
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.coarse_buffer(0), u_cc,
                                     static_cast<size_t>(S.kind_size((1u << dim) - 1u)) * sizeof(double),
                                     cudaMemcpyHostToDevice, plan->stream));
  const double* cs[3] = {dsol[0], dsol[1], dsol[2]};
  S.stage_skeleton(cs, u_cc ? S.coarse_buffer(0) : nullptr, seed, S.e_buffer(), plan->stream);
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(out, S.e_buffer(), static_cast<size_t>(S.fine_size()) * sizeof(double),
                                   cudaMemcpyDeviceToHost, plan->stream));
  ASDSM_CUDA_CHECK(cudaStreamSynchronize(plan->stream));
}
}  // namespace

int asdsm_build_skeleton(asdsm_plan* plan, const double* u_fc, const double* u_cf, const double* u_cc, int normalized,
                         uint64_t rng_seed, double* out) {
  return guarded([&] {
    if (plan->solver->mesh().dim != 2) throw AsdsmError(kInvalidKind, "build_skeleton is the 2D path; merge_3d handles 3D");
    if ((u_cc != nullptr) == (normalized != 0))
      throw AsdsmError(kInvalidKind, "coarse solution must be present exactly for unnormalized inputs");
    const double* sol[2] = {u_cf, u_fc};
    skeleton_call(plan, sol, u_cc, rng_seed, out);
  });
}

int asdsm_merge_3d(asdsm_plan* plan, const double* u_x, const double* u_y, const double* u_z, const double* u_ccc,
                   uint64_t rng_seed, double* out) {
  return guarded([&] {
    if (plan->solver->mesh().dim != 3) throw AsdsmError(kInvalidKind, "merge_3d is the 3D path");
    const double* sol[3] = {u_x, u_y, u_z};
    skeleton_call(plan, sol, u_ccc, rng_seed, out);
  });
}

int asdsm_fill_holes(asdsm_plan* plan, const double* skeleton, const double* b_fine, double* out) {
  return guarded([&] {
    Solver& S = *plan->solver;
    const Mesh& m = S.mesh();
    const i64 n = S.fine_size();
    // SkeletonNotHollow (solver.cpp:420-421): the input must vanish on every hole position
    for (i64 p = 0; p < n; ++p) {
      i64 q = p;
      bool hole = true;
      for (int a = 0; a < m.dim && hole; ++a) {
        hole = (static_cast<int>(q % m.nf[a]) + 1) % m.n[a] != 0;
        q /= m.nf[a];
      }
      if (hole && skeleton[p] != 0.0) throw AsdsmError(kSkeletonNotHollow, "fill_holes: skeleton has values inside holes");
    }
    const size_t nb = static_cast<size_t>(n) * sizeof(double);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.e_buffer(), skeleton, nb, cudaMemcpyHostToDevice, plan->stream));
    if (b_fine) ASDSM_CUDA_CHECK(cudaMemcpyAsync(S.r_buffer(1), b_fine, nb, cudaMemcpyHostToDevice, plan->stream));
    S.stage_fill(S.e_buffer(), b_fine ? S.r_buffer(1) : nullptr, plan->stream);
    ASDSM_CUDA_CHECK(cudaMemcpyAsync(out, S.e_buffer(), nb, cudaMemcpyDeviceToHost, plan->stream));
    ASDSM_CUDA_CHECK(cudaStreamSynchronize(plan->stream));
  });
}

}  // extern "C"
