#pragma once
#include "kernels.cuh"

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

}  // namespace asdsm_b200
