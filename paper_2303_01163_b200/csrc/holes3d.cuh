#pragma once
#include "kernels.cuh"

#include <vector>

namespace asdsm_b200 {

// Error-mode fill of 3D holes (fill_core, proj/src/solver.cpp:414-432) for the separable
// solver with line axis 2 and diagonalized axes 0, 1.
struct Hole3DArgs {
  int m[3];          // hole extents
  int n[3];          // refinement factors
  int nf[3];         // fine extents
  int nbox[3];       // holes per axis
  Stencil st;        // fine stencil
  const double* Wx;  // forward eigenvectors along x [k][i]
  const double* Wy;  // along y [l][j]
  const double* ipiv;  // Thomas [t][combo = k + m0 l]
  const double* cp;
  double line_left;
  double* faces;     // per hole: YA0,YA1 [t][l]; XB0,XB1 [t][k]; CH0,CH1 [l][k]
};

__host__ __device__ inline size_t hole3d_face_doubles(const Hole3DArgs& A) {  // per hole
  return 2 * static_cast<size_t>(A.m[2]) * A.m[1] + 2 * static_cast<size_t>(A.m[2]) * A.m[0] +
         2 * static_cast<size_t>(A.m[1]) * A.m[0];
}
void hole3d_prepare(const Hole3DArgs& A);  // shared-memory attribute, before any capture
void launch_hole3d_faces(const double* e, const Hole3DArgs& A, DevState* st, cudaStream_t s);
void launch_hole3d_thomas(double* modes, const Hole3DArgs& A, DevState* st, cudaStream_t s);

// One-kernel 3D error-mode fill (holes3d_fused.cu): same separable solve, faces + line solves +
// both back transforms per hole in shared memory, even/odd-split transforms.
struct H3Axis {    // one diagonalized axis of the hole
  int m, he, ho;   // points (= modes), even / odd mode counts
  int khe, kho;    // padded to multiples of 4
  int hrow, sh;    // half table: rows (pad8(he)) and row stride
};
struct H3Layout {  // shared memory, in doubles
  int tx, ty;      // half tables + sc + ci of x and y
  int ntx, nty;    // their sizes
  int faces;       // face transforms (SYM: YA, XB, CH; CAUSAL: CH0 + per-chunk ring / vectors)
  int x;           // resident planes [tc][rp][skx] + slack
  int xsize;
  int rp, skx;     // plane rows (even/odd l order, zero gaps), row stride
  int kxo, kyo;    // padded odd mode counts
  int tc;          // planes resident at once (SYM: all)
  int lg, lu;      // CAUSAL: thread (k, l0) owns the lines (k, l0 + lg u), u < lu
  size_t bytes;
};
struct Hole3DFusedArgs {
  int m[3], n[3], nf[3], nbox[3];
  Stencil st;
  const double* Hx;  // hole3d_half_table of x / y
  const double* Hy;
  H3Axis ax, ay;
  const double* ipiv;  // Thomas [t][combo = k + mx l]
  const double* cp;
  double line_left;
  H3Layout lay;
};
// Fills A.ax/ay/lay for the schedule (causal: line_right == 0); false if the hole does not fit.
bool hole3d_fused_plan(Hole3DFusedArgs& A, bool causal);
// Shared-memory half table of one axis from SepSolver::half (host copy).
std::vector<double> hole3d_half_table(const H3Axis& a, const std::vector<double>& half);
void hole3d_fused_prepare();
void launch_hole3d_fused(double* e, const Hole3DFusedArgs& A, bool causal, DevState* st, cudaStream_t s);

}  // namespace asdsm_b200
