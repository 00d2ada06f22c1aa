// B200 ASDSM solver context: the device-resident counterpart of the reference's
// SolverContext + asdsm_iterate (proj/include/asdsm/solver.hpp:114-163).
#pragma once
#include <cstdint>
#include <functional>
#include <cstdlib>
#include <string>
#include <vector>

#include "holes3d.cuh"
#include "kernels.cuh"
#include "merge3d.cuh"
#include "march.cuh"
#include "plan.hpp"
#include "sepsolve.cuh"
#include "varcoef.hpp"
#include "vthomas.cuh"
#include "slabstep2d.cuh"

namespace asdsm_b200 {

// IterateOptions (proj/include/asdsm/solver.hpp:56-68).
struct RunOptions {
  double tol = 1e-12;
  int max_iter = 20;
  int stagnation_window = 3;
  double stagnation_ratio = 0.99;
  double subsample = 0.0;
  std::uint64_t rng_seed = 0;
  bool sparse_residual = false;
};

std::uint64_t mix_seed(std::uint64_t base, std::uint64_t k);  // solver.cpp:88-96

class Solver {
 public:
  Solver(const Mesh& m, const double* alpha, const double* beta);
  // Variable coefficients (ProblemSpec with per-point alpha/beta): per-point stencils and
  // block-Thomas direct solves.
  Solver(const Mesh& m, const asdsm_cat::Problem& problem);
  bool separable_fallback() const { return separable_fallback_; }
  bool variable() const { return variable_; }
  Solver(const Solver&) = delete;
  Solver& operator=(const Solver&) = delete;

  const Mesh& mesh() const { return mesh_; }
  i64 fine_size() const { return g_fine_.size; }
  i64 slab_size(int a) const { return g_slab_[a].size; }
  i64 coarse_size() const { return g_coarse_.size; }

  // Right-hand-side bundle (RhsBundle, solver.hpp:37-42) + optional exact samples.
  // Pointers are host or device memory according to `on_device`.
  void set_bundle(const double* b_fine, const double* const* b_slab, const double* b_coarse, const double* exact,
                  bool on_device, cudaStream_t s);

  // Initial guess + up to max_iter error-mode corrections, all control on the device.
  void run(const RunOptions& o, cudaStream_t s);
  // IterateOptions::observer (solver.hpp:65): the solve launch by launch (no captured graph),
  // `after_record(k)` on the host after record k is enqueued (k = 0 first); it returns false to
  // stop enqueueing (the device state has stopped).  snapshot() reads the state in between.
  void run_observed(const RunOptions& o, cudaStream_t s, const std::function<bool(int)>& after_record);
  // history rows so far, and the current iterate / residual (host, nullable); returns nrec.
  int snapshot(std::vector<double>& rows, bool& active, double* u_out, double* r_out, cudaStream_t s);

  // After run(): history rows (k, res_l2, res_inf, err_max, err_l2, s_hat, wall_ms).
  int history(std::vector<double>& rows, int& stop_code, cudaStream_t s);
  // After run(): history rows, and the final iterate / residual to u_out / r_out (host or
  // device memory, nullable), enqueued together on `s` with a single synchronize.
  int fetch(std::vector<double>& rows, int& stop_code, double* u_out, double* r_out, cudaStream_t s);
  const double* u_current(cudaStream_t s) const;  // synchronizes to read the selector
  const double* r_current(cudaStream_t s) const;
  double* u_buffer(int i) { return u_[i]; }
  double* r_buffer(int i) { return r_[i]; }
  // The reference's public stages (solver.hpp:70-105, stages.cu) on device arrays of this plan's
  // mesh kinds: richardson_extrapolate, the coarse restriction choose_cross_points picks from
  // (cross_point_choice: 0 = u_cf, 1 = u_fc), spline_correct, build_skeleton / merge_3d (sol[a]:
  // the field on the kind coarse along a; u_cc null in error mode) and fill_holes (e: the
  // skeleton in, completed out; b null: zero right-hand side).
  void stage_richardson(const double* u1, const double* u2, const double* ucc, double* out, cudaStream_t s);
  void stage_restrict(const double* slab, int axis, double* out, cudaStream_t s);
  int cross_point_choice(std::uint64_t seed) const;
  void stage_spline_correct(const double* u, const double* ecc, int dense, double* out, cudaStream_t s);
  void stage_skeleton(const double* const* sol, const double* u_cc, std::uint64_t seed, double* out, cudaStream_t s);
  void stage_fill(double* e, const double* b, cudaStream_t s);
  double* slab_buffer(int a) { return sol_slab_[a]; }
  double* coarse_buffer(int i) { return i == 0 ? u_cc_ : i == 1 ? cc_e1_ : cc_e2_; }
  i64 kind_size(unsigned mask) const { return mask == 0 ? g_fine_.size : mask == (1u << mesh_.dim) - 1u ? g_coarse_.size : g_slab_[mask == 1u ? 0 : mask == 2u ? 1 : 2].size; }
  double* e_buffer() { return e_; }
  const double* b_fine() const { return b_; }

  // Single operations (for the function-level parity tests).
  void residual(const double* u, const double* b, double* r, cudaStream_t s);  // device pointers
  void error_guess(const double* r, std::uint64_t seed, double* e, cudaStream_t s);
  double optimal_scaling(const double* r, const double* e, cudaStream_t s);
  void initial_guess(double* u_out, std::uint64_t seed, cudaStream_t s);

  const MeshDev& mesh_dev() const { return md_; }

  // Component timing for the roofline (CUDA events on `s`, `reps` launches each, after a
  // run()).  Names/ms/bytes/flops per launch and launches per solve.
  struct Component {
    std::string name;
    double ms = 0, bytes = 0, flops = 0;
    int per_solve = 0;
  };
  std::vector<Component> profile(cudaStream_t s, int reps);

  // Launch count of the last run() (kernels of this library only).
  long long last_launches() const { return launches_; }
  // Kernels of the captured solve graph (demangled name, node count), from the graph's own
  // kernel nodes: what a solve actually launches (tests assert the intended variant ran).
  const std::vector<std::pair<std::string, int>>& graph_kernels() const { return graph_kernels_; }
  ~Solver();

 private:
  void reset_state(const RunOptions& o, cudaStream_t s);
  void enqueue_run(const RunOptions& o, cudaStream_t s, const std::function<bool(int)>* after_record = nullptr);
  void prepare_run(const RunOptions& o, cudaStream_t s);
  void run_graph(const RunOptions& o, cudaStream_t s);
  void smooth_guess(double* out, cudaStream_t s);
  void error_mode_guess(const double* r0, const double* r1, int k, double* out, cudaStream_t s);
  void skeleton(const double* const* sol, const double* u_cc, const int* coin, double* out, cudaStream_t s);
  // stage: kFillAll, or (2D two-kernel hole path, for per-component timing) kFillLines = ring rhs +
  // mode-line solves only, kFillBack = the back transform only
  enum { kFillLines = 1, kFillBack = 2, kFillAll = 3 };
  void fill(double* e, const double* b, cudaStream_t s, int stage = kFillAll);
  BoxArray hole_array(double* p) const;
  BoxArray kind_array(const KindGeom& g, double* p) const;

  void init(const asdsm_cat::Problem* varprob);
  // constant coefficients whose boxes the separable solvers cannot take (an eigenvector
  // scaling too ill-conditioned on every candidate transform axis -- strong advection over a
  // long box -- or complex modes on two diagonalized axes): the same operator as constant
  // per-point fields on the block-Thomas path (no CPU fallback, no Unsupported)
  asdsm_cat::Problem const_fields_{};
  bool separable_fallback_ = false;
  void solve_box(int which, double* data, cudaStream_t s);
  void march_launch(int mode, struct MarchArgs A, cudaStream_t s);  // variable mode: 0..2 slab, 3 coarse, 4 holes
  Mesh mesh_;
  bool variable_ = false;
  double* coef_fine_ = nullptr;
  BTDev bt_[5]{};
  double alpha_[3] = {0, 0, 0}, beta_[3] = {0, 0, 0};
  MeshDev md_{};
  KindGeom g_fine_, g_slab_[3], g_coarse_;
  FineGeom fg_{};
  Stencil st_fine_, st_slab_[3], st_coarse_;
  SepSolver sep_slab_[3], sep_coarse_, sep_hole_;
  DeviceAlloc dev_;
  double* u_[2] = {nullptr, nullptr};
  double* r_[2] = {nullptr, nullptr};
  double* b_ = nullptr;
  double* e_ = nullptr;
  double* exact_ = nullptr;
  bool has_exact_ = false;
  double* b_slab_[3] = {nullptr, nullptr, nullptr};
  double* rhs_slab_[3] = {nullptr, nullptr, nullptr};
  double* sol_slab_[3] = {nullptr, nullptr, nullptr};
  double* b_coarse_ = nullptr;
  double* u_cc_ = nullptr;
  double* cc_e1_ = nullptr;
  double* cc_e2_ = nullptr;
  double* spl_m1_ = nullptr;
  double* spl_m2_ = nullptr;
  Merge3DArgs m3_{};
  bool fast2d_ = false;          // fused 2D slab/skeleton/hole path
  double* slab_modes_[2] = {nullptr, nullptr};
  double* stations_[2] = {nullptr, nullptr};  // residual on the slab stations (per residual buffer)
  double* sp_basis_[2] = {nullptr, nullptr};    // skeleton-correction basis per axis (nf x nc)
  bool step2d_ = false;
  double* skel_line_[2] = {nullptr, nullptr};   // slab step outputs: normalized station lines
  double* skel_corr_ = nullptr;                 //   and the cross-point corrections
  bool ring_from_lines_ = false;                // fill(): holes evaluate + write the skeleton
  double* hole_ring_ = nullptr;                 // 2D large holes: [hole][2 m1 + 2 m0] ring + row transforms
  // 2D large holes, error mode: strip split (holes2d.cuh launch_hole2d_sep_rows) -- p strips of
  // w columns per hole between p - 1 separator columns, each solved as a hole of its own
  int strip_p_ = 0;
  SepSolver sep_strip_{};
  double* strip_ring_ = nullptr;
  // the separators from one GEMM with the separator response matrix K ((p-1) m1 x (2 m1 + 2 m0),
  // column-major, built at plan creation; holes2d.cuh): sep = K ring, on cuBLAS
  double* sep_K_ = nullptr;
  double* sep_C_ = nullptr;  // [hole][(p-1) m1]
  int sep_rows_ = 0, sep_cols_ = 0;
  void* blas_ = nullptr;     // cublasHandle_t
  void* blas_ws_ = nullptr;  // its workspace (set explicitly: no allocation during stream capture)
  void build_separator_matrix();
  bool dots_update_ok_ = false;                 // kMarchDotsUpdate on (ASDSM_DOTS_UPDATE=1) and applicable
  // optimal-step dot products over the skeleton rows only (ASDSM_FULL_DOTS=1: every row)
  bool skel_dots_ = std::getenv("ASDSM_FULL_DOTS") == nullptr;                          // one-launch slab step (slabstep2d.cu) eligible
  double* sp_tab_[2] = {nullptr, nullptr};
  double* seg1_ = nullptr;
  double* seg2_ = nullptr;
  double* faces3d_ = nullptr;  // 3D fused fill: transformed hole faces
  Hole3DFusedArgs h3f_{};      // 3D one-kernel fill (holes3d_fused.cu), when the hole fits
  bool h3f_ok_ = false;
  bool h3f_causal_ = false;
  std::vector<long long> skel_rows_;  // ascending skeleton rows (subsample > 0), built lazily
  long long* sub_rows_ = nullptr;     // per-iteration sorted subsets, [k][m]
  size_t sub_cap_ = 0;
  int sub_m_ = 0;
  Skel2DArgs skel2d_args(const double* const* sol, const double* u_cc, const int* coin, double* out);
  SlabStep2DArgs slabstep2d_args(const int* coin, double* out) const;
  void* scratch0_ = nullptr;
  void* scratch1_ = nullptr;
  void* slab_scr_[3][2] = {{nullptr, nullptr}, {nullptr, nullptr}, {nullptr, nullptr}};  // 3D: slabs 1, 2
  cudaStream_t aux_[2] = {nullptr, nullptr};  // 3D: streams of slabs 1 and 2
  cudaEvent_t ev_[3] = {nullptr, nullptr, nullptr};
  double* partials_ = nullptr;
  DevState* state_ = nullptr;
  double* history_ = nullptr;
  int history_cap_ = 0;
  DevState* host_state_ = nullptr;  // pinned staging of the state and history for fetch()
  double* host_hist_ = nullptr;
  int host_hist_cap_ = 0;
  int* coins_ = nullptr;
  int coins_cap_ = 0;
  RunOptions last_opts_{};
  double cell_ = 1.0;
  long long launches_ = 0;
  cudaGraphExec_t graph_exec_ = nullptr;
  RunOptions graph_opts_{};
  bool graph_has_exact_ = false;
  std::vector<std::pair<std::string, int>> graph_kernels_;  // CtrlArgs.has_exact and the exact_ pointer are baked into the graph
  long long graph_launches_ = 0;
};

}  // namespace asdsm_b200
