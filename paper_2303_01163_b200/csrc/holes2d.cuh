#pragma once
#include "kernels.cuh"

namespace asdsm_b200 {

struct Hole2DArgs {
  int m0, m1;        // hole extents (x modes, y rows)
  int n0, n1;        // refinement factors
  int nf0, nf1;      // fine extents
  int nbox0, nbox1;  // holes per axis (nc + 1)
  int kb;            // modes per CTA
  Stencil st;        // fine stencil
  const double* Wt;  // forward eigenvectors along x, transposed: Wt[i*m0 + k] = W[k][i]
  const double* half;  // even/odd half sine table + row scalings along x (SepSolver::half)
  // error mode after the one-launch slab step: the ring is evaluated here from the normalized
  // station-line values + the spline of the cross-point corrections (else read from the fine
  // array), and the hole writes the skeleton lines it owns (its left column and bottom row)
  const double* skel_line0;  // [nc0][nf1]
  const double* skel_line1;  // [nc1][nf0]
  const double* corr;        // E1 then E2 (nc0*nc1 each)
  const double* basis0;      // spline_basis_table of axis 0 [nf0][nc0]
  const double* basis1;      // [nf1][nc1]
  int nc0, nc1;
  const double* ipiv;  // Thomas pivots [j][k]
  const double* cp;    // Thomas upper factors [j][k]
  double line_left, line_right;
  int y_in_smem;     // park the forward sweep in shared memory (else in the mode buffer)
  int tables_in_smem;  // bulk-load this CTA's slices of Wt / ipiv / cp into shared memory first
};

// fused whole-hole kernel (ring rhs + sweeps + DMMA back transform) for holes up to 128^2
constexpr size_t kHole2DFusedMaxSmem = 220 * 1024;
// shared row stride of the fused kernel's tiles (compile time, so row offsets are immediates):
// = 12 (mod 16) doubles, so the 8 rows x 4 k of an m8n8k4 fragment load hit distinct bank
// pairs; holes with up to 108 modes along x use the fused kernel
constexpr int kHole2DFusedStride = 108;
size_t hole2d_fused_smem_bytes(int m0, int m1);
bool hole2d_fused_fits(int m0, int m1);
// b == nullptr: error mode (ring-only rhs); else smooth mode, rhs = b - A_hs skeleton
void launch_hole2d_fused(double* e, const Hole2DArgs& A, const double* b, DevState* state, cudaStream_t s);
size_t hole2d_smem_bytes(int m0, int m1, int kb, bool y_in_smem, bool tables_in_smem = false);
void hole2d_prepare(size_t smem);
void launch_hole2d_fwd_thomas(const double* e, double* modes, const Hole2DArgs& A, DevState* state, cudaStream_t s);
// Large holes, error mode, as two launches over a per-hole ring buffer ([hole][2 m1 + 2 m0]:
// fL, fR, fB, fT): (1) one CTA per hole forms the ring; (2) one warp per (hole, mode k) forms the
// two full row transforms of mode k (coalesced row of W, warp-shuffle sums), builds the mode
// line and solves it with the warp partition method (SepSolver::part tables), writing modes as
// [hole][k][j] (j contiguous: the back transform reads it with in_es = m1).
struct Hole2DPartArgs {
  const double* W;     // forward eigenvectors along x, [k][i] (row k contiguous)
  const double* part;  // SepSolver::part of the hole solver, stride pstride per mode
  int pstride, seg, P, last;
  double* ring;        // [hole][2 m1 + 2 m0]
};
bool hole2d_part_supported(int seg);
void launch_hole2d_ring(const double* e, const Hole2DArgs& A, const Hole2DPartArgs& P, DevState* state,
                        cudaStream_t s);
void launch_hole2d_part(double* modes, const Hole2DArgs& A, const Hole2DPartArgs& P, DevState* state, cudaStream_t s);

// Strip split of large holes (error mode): once the mode lines of a hole are solved
// (modes[hole][k][j]), its solution on the p - 1 separator columns i_s = s (w + 1) - 1 is
// v(i_s, j) = sum_k V[i_s][k] modes[k][j]: a (p - 1) x m0 by m0 x m1 product per hole, written
// into the fine array.  The p strips of w = (m0 + 1) / p - 1 columns between separators are then
// holes of their own (Dirichlet data: skeleton and separators) with w-point transforms, so the
// back transform costs w instead of m0 per point.
void launch_hole2d_sep_rows(const double* modes, const double* V, double* e, const Hole2DArgs& A, int p,
                            DevState* state, cudaStream_t s, double* dense = nullptr);
// The separator values can also come from one GEMM per iteration: the solution on the separators
// is linear in the hole's ring right-hand side (2 m1 + 2 m0 values, holes2d ring layout), so
// sep = K ring with K the (p-1) m1 x (2 m1 + 2 m0) separator response matrix -- the same for
// every hole (congruent holes), built once at plan creation by running the mode-line and
// separator kernels on unit rings (dense != nullptr: [hole][s][j] output instead of the fine
// array).  launch_hole2d_sep_scatter writes the GEMM's [hole][s][j] columns into the fine array.
void launch_hole2d_sep_scatter(const double* sep, double* e, const Hole2DArgs& A, int p, DevState* state,
                               cudaStream_t s);

}  // namespace asdsm_b200
