// ASDSM iteration kernels (declarations).  See kernels.cu.
#pragma once
#include "plan.hpp"

#include <vector>

namespace asdsm_b200 {

constexpr int kRedBlocks = 4 * kNumSms;  // fixed grid => deterministic reduction order
constexpr int kRedStride = 65536;         // partials[slot * kRedStride + block], blocks <= kRedStride
constexpr int kRedThreads = 256;

// Device-resident iteration state (the reference's IterationState scalars,
// proj/include/asdsm/solver.hpp:49-54, plus the buffer selector).
struct DevState {
  int cur;       // which of u[0]/u[1], r[0]/r[1] is the current iterate
  int active;    // 0 once a stop rule fired
  int have_e;    // error guess exists (no ZeroNormSolution)
  int stop;      // 0 running, 1 tol, 2 stagnation, 3 max_iter
  int nrec;      // history rows written
  unsigned red_counter;  // blocks finished in the current folded reduction
  double res_l2, res_inf, err_max, err_l2;
  double s;                      // step of the current iteration
  double num, den;               // <r, Ae>, <Ae, Ae>
  double next_l2, next_inf, next_errmax, next_errl2;
  double slab_norm[3];
  double stop_at;                // tol * ||b||_2 (or tol when b == 0)
  double b_l2;
  double t0_ns;                  // %globaltimer at state init (history wall_ms origin)
  double num_sub, den_sub;       // subsampled <r,Ae>, <Ae,Ae> (subsample > 0)
  double s_full;                 // all-rows step, for the residual-growth retry
  int retry;                     // subsampled step grew the residual: second update pending
  unsigned gen;                  // grid-barrier generation (fused dots + update pass)
};

struct FineGeom {
  int dim;
  int ext[3];
  i64 stride[3];
  i64 size;
};

struct MeshDev {  // mesh scalars the skeleton kernels need
  int dim;
  int nf[3], nc[3], n[3];
  double h[3];
};

struct CtrlArgs;

// Reductions: partials[slot * kRedBlocks + block]; slots: 0 sum, 1 max, 2 sum, 3 max.  With a
// non-null `ctrl`, the last block to finish reduces the partials and applies the control op.
void launch_stencil(int dim, bool update, const double* u0, const double* u1, const double* e, const double* b,
                    double* uo0, double* uo1, double* ro0, double* ro1, const double* exact, const FineGeom& g,
                    const Stencil& st, double* partials, DevState* state, cudaStream_t s,
                    const CtrlArgs* ctrl = nullptr, double* history = nullptr);
void launch_ae_dots(int dim, const double* e, const double* r0, const double* r1, const FineGeom& g,
                    const Stencil& st, double* partials, DevState* state, cudaStream_t s,
                    const CtrlArgs* ctrl = nullptr, double* history = nullptr);
void launch_gather(const double* src0, const double* src1, double* dst, const MeshDev& m, unsigned mask,
                   i64 count, DevState* state, cudaStream_t s);
void launch_norm_sq(const double* x, i64 n, double* partials, DevState* state, cudaStream_t s,
                    const CtrlArgs* ctrl = nullptr, double* history = nullptr);
void launch_divide(double* x, i64 n, const double* divisor, DevState* state, cudaStream_t s);

// Device-side state initialization (capturable in a CUDA graph; no host memcpy).
void launch_state_init(DevState* state, int active, int have_e, cudaStream_t s);
void launch_spin(double us, cudaStream_t s);
// Current iterate into u[0]/r[0] (copy when the selector is 1, then selector = 0): a fetch can
// enqueue its device-to-host copies without reading the selector on the host first.
void launch_publish(DevState* state, double* u0, const double* u1, double* r0, const double* r1, i64 n,
                    cudaStream_t s);

// Final reductions + control (single CTA).
enum CtrlOp {
  kCtrlResidualK0 = 0,   // res norms of r0 (+ err) -> state, record row 0
  kCtrlSlabNorm = 1,     // slot sum -> slab_norm[which]; have_e &= norm > 0
  kCtrlStep = 2,         // num/den -> s
  kCtrlAccept = 3,       // next norms; accept/revert; record row k; stop rules
  kCtrlInit = 4,         // ||b||_2 -> stop_at = tol * (||b|| > 0 ? ||b|| : 1)
  kCtrlSlabNorms2 = 5,   // slot 0 / slot 2 sums -> slab_norm[0], slab_norm[1]; have_e
  kCtrlSetStep = 6,      // profiling only: s = CtrlArgs::cell
  kCtrlSubDots = 7,      // subsampled dots -> num_sub, den_sub
  kCtrlAccept2 = 8,      // outcome of the all-rows retry update (subsample > 0)
};
struct CtrlArgs {
  int op;
  int which;
  int k;
  int has_exact;
  double cell;          // prod fine steps (err_l2 weight)
  double tol_growth;    // 1 + 1e-12
  int stagnation_window;
  double stagnation_pow;  // ratio^window
  int max_iter;
  double tol;
  int subsample;        // subsample > 0: step from the seeded row subset, all-rows retry
};
void launch_ctrl(const CtrlArgs& a, const double* partials, DevState* state, double* history, cudaStream_t s);

// 2D skeleton (solver.cpp:154-196) and fill (solver.cpp:414-432).
struct Skel2DArgs {
  MeshDev m;
  const double* u_fc;   // slab coarse along y: ext (nf0, nc1)
  const double* u_cf;   // slab coarse along x: ext (nc0, nf1)
  const double* u_cc;   // smooth mode coarse solution, or null
  const int* coin;      // error mode: coin[0] == 0 -> take P(u_cf), else P(u_fc)
  double* e1;           // cc-level corrections (nc0*nc1)
  double* e2;
  double* m1;           // spline second derivatives, nc1 lines x (nc0+2)
  double* m2;           // nc0 lines x (nc1+2)
  double* out;          // fine array: skeleton points written
  const double* norm_fc;  // error mode: ||u_fc||_2 (values are divided by it, solver.cpp:79-84), else null
  const double* norm_cf;
  // fast path (coarse counts <= 62): data-independent spline terms precomputed on the host
  // per axis [x (nc+2) | hl | hr | w | diag | upper (nc each)], and per-line segment
  // coefficients (y_c, c1, c2, c3) x (nc+1) written by the cc/spline phase.
  const double* sp_tab[2];
  double* seg1;  // nc1 lines along x
  double* seg2;  // nc0 lines along y
};
void launch_skeleton2d(const Skel2DArgs& a, DevState* state, cudaStream_t s);
// fast path pieces: cross values + spline segment coefficients (one CTA), skeleton write
void launch_skel2d_ccspline_fast(const Skel2DArgs& a, DevState* state, cudaStream_t s);
void launch_skel2d_write_fast(const Skel2DArgs& a, DevState* state, cudaStream_t s);
// host: the data-independent spline terms of one axis (bitwise the reference's values)
std::vector<double> spline_axis_table(int nc, int n, double h);
// host: skeleton-correction basis of one axis, B[i][I] (nf x nc) -- see kernels.cu
std::vector<double> spline_basis_table(int nc, int n, double h, int nf);

void launch_hole_rhs(int dim, double* e, const double* b, const FineGeom& g, const Stencil& st, const MeshDev& m,
                     DevState* state, cudaStream_t s);

// subsample > 0: <r, Ae>, <Ae, Ae> over a sorted list of skeleton rows (solver.cpp:462-481),
// folded into kCtrlSubDots.
void launch_subsample_dots(int dim, const long long* rows, int nrows, const double* e, const double* r0,
                           const double* r1, const FineGeom& g, const Stencil& st, double* partials,
                           DevState* state, double* history, cudaStream_t s, const double* coef = nullptr);

// Dense coarse solve x = Ainv b (small), single CTA.
void launch_dense_matvec(const double* Ainv, const double* b, double* x, int n, DevState* state, cudaStream_t s);

}  // namespace asdsm_b200

namespace asdsm_b200 {
// Projector index maps (build_projector, proj/src/mesh.cpp:210-256) and the holes-kind
// order (hole_blocks, mesh.cpp:258-305), generated on the device.
void launch_projector_map(const MeshDev& m, unsigned from_mask, unsigned to_mask, long long* out, i64 count,
                          cudaStream_t s);
void launch_hole_map(const MeshDev& m, long long* out, i64 count, cudaStream_t s);
}  // namespace asdsm_b200
