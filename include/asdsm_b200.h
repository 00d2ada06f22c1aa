/*
 * asdsm_b200.h -- C-ABI of the B200-native ASDSM solver (libasdsm_b200.so).
 *
 * Plain pointers and sizes only; no torch or CUDA types in any signature (streams are
 * passed as void*).  Each entry point names the reference interface it replaces
 * (reference: proj/include/asdsm/*.hpp of arxiv/paper_2303_01163).  Errors are returned as
 * status codes that mirror the reference's exception classes (errors.hpp:8-66); the
 * message of the last failure on the calling thread is available from asdsm_last_error().
 *
 * Array layouts are the reference's: every mesh kind is linearized axis-0 fastest over
 * 1-based interior indices (mesh.hpp:72-75), the holes kind block by block (mesh.hpp:150-154).
 */
#ifndef ASDSM_B200_H
#define ASDSM_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ASDSM_B200_ABI_VERSION 4

/* Status codes <-> errors.hpp exception classes. */
enum asdsm_status {
  ASDSM_OK = 0,
  ASDSM_ERROR = 1,               /* asdsm::Error                               */
  ASDSM_DIVISIBILITY_ERROR = 2,  /* asdsm::DivisibilityError  (errors.hpp:15) */
  ASDSM_DEGENERATE_ERROR = 3,    /* asdsm::DegenerateError    (errors.hpp:21) */
  ASDSM_INDEX_OUT_OF_RANGE = 4,  /* asdsm::IndexOutOfRange    (errors.hpp:25) */
  ASDSM_NOT_A_SUBMESH = 5,       /* asdsm::NotASubmesh        (errors.hpp:31) */
  ASDSM_INVALID_KIND = 6,        /* asdsm::InvalidKind        (errors.hpp:36) */
  ASDSM_DIMENSION_MISMATCH = 7,  /* asdsm::DimensionMismatch  (errors.hpp:40) */
  ASDSM_SINGULAR_MATRIX = 8,     /* asdsm::SingularMatrix     (errors.hpp:44) */
  ASDSM_SKELETON_NOT_HOLLOW = 9, /* asdsm::SkeletonNotHollow  (errors.hpp:49) */
  ASDSM_ZERO_NORM_SOLUTION = 10, /* asdsm::ZeroNormSolution   (errors.hpp:55) */
  ASDSM_UNKNOWN_EXAMPLE = 11,    /* asdsm::UnknownExample     (errors.hpp:59) */
  ASDSM_NO_EXACT_SOLUTION = 12,  /* asdsm::NoExactSolution    (errors.hpp:63) */
  ASDSM_UNSUPPORTED = 13,        /* configuration outside the B200 path's scope */
  ASDSM_CUDA_FAILURE = 14        /* CUDA runtime failure (no GPU, OOM, ...)     */
};

/* Stop reasons of IterationState::stop_reason (solver.hpp:53). */
enum asdsm_stop { ASDSM_STOP_TOL = 1, ASDSM_STOP_STAGNATION = 2, ASDSM_STOP_MAX_ITER = 3 };

typedef struct asdsm_plan asdsm_plan;       /* SolverContext (solver.hpp:114-155), device-resident */
typedef struct asdsm_problem asdsm_problem; /* ProblemSpec (fdm.hpp:18-30), host-side catalogue   */

/* IterateOptions (solver.hpp:56-68). */
typedef struct {
  double tol;               /* relative to ||b||_2 (absolute when b == 0); default 1e-12 */
  int32_t max_iter;         /* default 20                                                */
  int32_t stagnation_window;/* 0 disables; default 3                                     */
  double stagnation_ratio;  /* default 0.99                                              */
  double subsample;         /* fraction of skeleton rows for the step length; 0 = all     */
  uint64_t rng_seed;        /* default 0                                                 */
  int32_t sparse_residual;  /* evaluate residual updates on skeleton rows only; default 0 */
} asdsm_iterate_options;

const char* asdsm_last_error(void);
int asdsm_abi_version(void);
void asdsm_default_options(asdsm_iterate_options* o);

/* ---- problems (problems.hpp:20 make_problem, example_mesh; fdm.hpp:44 assemble_rhs) ---- */
/* Reference example `example` (1..4), `setting` (1..2): problems.cpp:114-141. */
int asdsm_problem_example(int example, int setting, asdsm_problem** out);
/* BASELINE.json config id (0..4) with its seeded synthetic source. */
int asdsm_problem_config(int config_id, uint64_t seed, asdsm_problem** out);
/* A caller-defined ProblemSpec (fdm.hpp:17-30: dim, time_dependent, alpha/beta per spatial
 * axis, source, boundary, optional exact -- the reference's ScalarField callables) as C
 * callbacks, each with its own context pointer.  A field is evaluated at a point x[0..dim-1]
 * (the last coordinate is t when time_dependent), at the sampling points of the reference's
 * assembly (fdm.cpp:63-171), on host threads during plan creation and right-hand-side assembly
 * only -- never during a solve; fields must be pure (thread-safe).  alpha/beta entries past the
 * spatial axes are ignored (may be NULL); exact may be NULL.  The problem keeps the pointers:
 * contexts must outlive it.  Plans made from it take the separable constant-coefficient solvers
 * when every fine-node sample of alpha_a and beta_a is the same value, the per-point
 * (variable-coefficient) path otherwise -- the operator is the reference's either way. */
typedef double (*asdsm_field_fn)(const double* x, void* ctx);
typedef struct {
  asdsm_field_fn fn;
  void* ctx;
} asdsm_field;
typedef struct {
  int32_t dim;            /* 2 or 3 */
  int32_t time_dependent; /* last axis is t (backward difference; boundary = initial data) */
  asdsm_field alpha[3];   /* diffusion per spatial axis, positive */
  asdsm_field beta[3];    /* advection per spatial axis */
  asdsm_field source;
  asdsm_field boundary;
  asdsm_field exact;      /* fn NULL: no exact solution attached */
} asdsm_problem_spec;
int asdsm_problem_create(const asdsm_problem_spec* spec, asdsm_problem** out);
void asdsm_problem_destroy(asdsm_problem* p);
/* dim, time-dependence, constant coefficients (alpha/beta have 3 entries), exact available.
 * A caller-defined problem reports constant_coeffs = 0: plans decide it from their samples. */
int asdsm_problem_info(const asdsm_problem* p, int* dim, int* time_dependent, int* constant_coeffs,
                       double* alpha, double* beta, int* has_exact);
/* Mesh of a BASELINE config (fine/coarse counts, 3 entries each) and its iteration budget. */
int asdsm_config_mesh(int config_id, int* dim, int* fine_counts, int* coarse_counts, int* time_axis,
                      int* iterations);
/* assemble_rhs (fdm.hpp:44-46) on the tensor kind with coarse mask `mask`, host output. */
int asdsm_assemble_rhs(const asdsm_problem* p, int dim, const int* fine_counts, const int* coarse_counts,
                       int time_axis, unsigned mask, double* out);
/* exact solution samples on the fine mesh (problems.hpp:29 error_norms' samples). */
int asdsm_sample_exact(const asdsm_problem* p, int dim, const int* fine_counts, const int* coarse_counts,
                       int time_axis, double* out);

/* ---- plan (MeshConfig::create mesh.hpp:68 + SolverContext ctor solver.hpp:116) ---------- */
/* Constant per-axis coefficients alpha[3], beta[3] (spatial axes; time axis ignored). */
int asdsm_plan_create(int dim, const int* fine_counts, const int* coarse_counts, int time_axis,
                      const double* alpha, const double* beta, asdsm_plan** out);
/* Plan for a catalogue problem: constant coefficients take the separable fast solvers;
 * variable coefficients (fdm.hpp:18-30 ProblemSpec with per-point alpha/beta) are sampled on
 * the host as assemble_operator does (fdm.cpp:63-126) and solved with block Thomas. */
int asdsm_plan_create_problem(const asdsm_problem* problem, int dim, const int* fine_counts,
                              const int* coarse_counts, int time_axis, asdsm_plan** out);
int asdsm_plan_is_variable(const asdsm_plan* plan);
void asdsm_plan_destroy(asdsm_plan* plan);
/* MeshConfig::point_count (mesh.hpp:72) for a tensor kind (coarse mask) or the holes kind. */
int asdsm_point_count(const asdsm_plan* plan, unsigned coarse_mask, int holes, int64_t* out);
/* build_projector(...).index_map() (mesh.hpp:148): map from kind `from_mask` to kind
 * `to_mask` (or the holes kind when to_holes != 0); computed on the GPU; host output. */
int asdsm_projector_map(asdsm_plan* plan, unsigned from_mask, unsigned to_mask, int to_holes, int64_t* out);

/* RhsBundle (solver.hpp:37-42) + optional exact samples (nullable); host or device memory.
 * b_slab[a] lives on the kind coarse along axis a.  Returns after the copies completed; device
 * sources must be complete when it is called (synchronize their producer first). */
int asdsm_set_bundle(asdsm_plan* plan, const double* b_fine, const double* const* b_slab,
                     const double* b_coarse, const double* exact, int on_device);
/* Same, enqueued on `stream` (cudaStream_t as void*, NULL = the plan's stream) without a host
 * synchronize: ordered after the caller's producer work on `stream` and before a following
 * asdsm_iterate_async on the same stream.  Host sources must stay valid (and pinned for
 * overlap) until the stream reaches the copies. */
int asdsm_set_bundle_async(asdsm_plan* plan, const double* b_fine, const double* const* b_slab,
                           const double* b_coarse, const double* exact, int on_device, void* stream);

/* asdsm_iterate (solver.hpp:161-163).  Host outputs (all nullable): history rows of
 * (k, res_l2, res_inf, err_max, err_l2, s_hat, wall_ms), the final iterate u and residual r. */
int asdsm_iterate(asdsm_plan* plan, const asdsm_iterate_options* opts, double* history, int* nrec,
                  int* stop_code, double* u_out, double* r_out);
/* One call from host buffers to host results: asdsm_set_bundle (host memory) + asdsm_iterate, the
 * uploads, the solve and the downloads ordered on the plan's stream with a single synchronize
 * (the host buffers are free again when it returns).  The reference's
 * asdsm_iterate(problem, config, options) on a prebuilt SolverContext (solver.hpp:161-163). */
int asdsm_solve(asdsm_plan* plan, const double* b_fine, const double* const* b_slab, const double* b_coarse,
                const double* exact, const asdsm_iterate_options* opts, double* history, int* nrec,
                int* stop_code, double* u_out, double* r_out);
/* asdsm_iterate with IterateOptions::observer (solver.hpp:65-66): `observer` is called after each
 * recorded iteration (k = 0 first) with the history rows so far (7 doubles each, as
 * asdsm_iterate), the current iterate u and residual r (n fine values each; host arrays valid
 * during the call) -- the reference's IterationState at that point.  The solve runs launch by
 * launch with one stream synchronize per iteration instead of the captured graph (same
 * arithmetic, so the same results); the final outputs are asdsm_iterate's. */
typedef void (*asdsm_observer_fn)(const double* history, int nrec, const double* u, const double* r, int64_t n,
                                  void* ctx);
int asdsm_iterate_observed(asdsm_plan* plan, const asdsm_iterate_options* opts, asdsm_observer_fn observer, void* ctx,
                           double* history, int* nrec, int* stop_code, double* u_out, double* r_out);
/* Same solve fully on `stream` (cudaStream_t as void*, NULL = legacy): no host sync. */
int asdsm_iterate_async(asdsm_plan* plan, const asdsm_iterate_options* opts, void* stream);
/* After asdsm_iterate_async: history/outputs to host (synchronizes the stream). */
int asdsm_fetch(asdsm_plan* plan, void* stream, double* history, int* nrec, int* stop_code, double* u_out,
                double* r_out);
/* Device pointer of the current iterate (valid until the next call on the plan). */
int asdsm_device_solution(asdsm_plan* plan, void* stream, const double** u_dev);
/* Kernels this library launched during the last iterate call. */
int64_t asdsm_last_launch_count(const asdsm_plan* plan);
/* The kernels of the plan's captured solve graph: "name<TAB>nodes<NEWLINE>" per kernel
 * (demangled), NUL-terminated, truncated to len-1 bytes.  Empty before the first graph solve. */
int asdsm_plan_kernels(const asdsm_plan* plan, char* buf, int64_t len);

/* The plan's own stream (cudaStream_t as void*). */
void* asdsm_plan_stream(asdsm_plan* plan);
/* Component timing after an iterate call: each component of one ASDSM iteration launched
 * `reps` times between CUDA events on `stream`; per launch: ms, algorithmic bytes and
 * flops, and launches per solve.  names: 64 chars per component. */
int asdsm_profile_components(asdsm_plan* plan, void* stream, int reps, int max_components, char* names, double* ms,
                             double* bytes, double* flops, int* per_solve, int* count);

/* ---- single operations for parity tests (host arrays) ------------------------------- */
int asdsm_residual(asdsm_plan* plan, const double* u, const double* b, double* r);     /* fdm.hpp:50 */
int asdsm_initial_guess(asdsm_plan* plan, double* u_out);                              /* solver.hpp:132 (smooth) */
int asdsm_error_guess(asdsm_plan* plan, const double* r, uint64_t seed, double* e_out); /* solver.hpp:135 */
int asdsm_optimal_scaling(asdsm_plan* plan, const double* r, const double* e, double* s_out); /* solver.hpp:109 */

/* ---- public solver stages (solver.hpp:70-105; host arrays of this plan's mesh kinds) ------
 * Single device operations with the reference's operation order (bitwise its results, except
 * fill_holes whose direct solves round differently) and argument checks.  They reuse the plan's
 * work buffers: a following asdsm_iterate re-initializes them. */
/* richardson_extrapolate (solver.hpp:72-73): u1_cc + u2_cc - u_cc on the coarse mesh. */
int asdsm_richardson_extrapolate(asdsm_plan* plan, const double* u1_cc, const double* u2_cc, const double* u_cc,
                                 double* out);
/* choose_cross_points (solver.hpp:78-79, 2D): the coarse restriction of u_cf (coarse along x) or
 * u_fc (coarse along y) picked by mt19937_64(rng_seed). */
int asdsm_choose_cross_points(asdsm_plan* plan, const double* u_fc, const double* u_cf, uint64_t rng_seed,
                              double* out);
/* spline_correct (solver.hpp:84-85, 2D): u_aniso (on the kind coarse along 1 - dense_axis) plus
 * the zero-clamped natural cubic spline of the coarse correction e_cc along dense_axis. */
int asdsm_spline_correct(asdsm_plan* plan, const double* u_aniso, const double* e_cc, int dense_axis, double* out);
/* build_skeleton (solver.hpp:90-91, 2D; SkeletonInputs solver.hpp:23-29): u_cc given exactly when
 * normalized == 0 (else InvalidKind); fine-mesh output, holes exactly zero. */
int asdsm_build_skeleton(asdsm_plan* plan, const double* u_fc, const double* u_cf, const double* u_cc, int normalized,
                         uint64_t rng_seed, double* out);
/* merge_3d (solver.hpp:98-100): u_x/u_y/u_z on the kinds coarse along x/y/z, u_ccc nullable
 * (error mode: seeded slab choices). */
int asdsm_merge_3d(asdsm_plan* plan, const double* u_x, const double* u_y, const double* u_z, const double* u_ccc,
                   uint64_t rng_seed, double* out);
/* fill_holes (solver.hpp:104-105): the skeleton completed by the hole solves against b_fine
 * (nullable: zero); SKELETON_NOT_HOLLOW when the input has values on hole positions. */
int asdsm_fill_holes(asdsm_plan* plan, const double* skeleton, const double* b_fine, double* out);

#ifdef __cplusplus
}
#endif
#endif /* ASDSM_B200_H */
