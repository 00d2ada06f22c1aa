#pragma once
#include "kernels.cuh"

namespace asdsm_b200 {

struct BTDev {
  int dim, L, B, nb;
  int ext[3];
  const double* dinv;  // [box][j][k*B+i]
  const double* lo;    // [box][j][i]
  const double* up;
};

// In-place block-Thomas solve of every box of `arr` (one CTA per box).
void launch_block_thomas(const BTDev& T, const BoxArray& arr, DevState* st, cudaStream_t s);

// Hole rhs with per-point coefficients (coef[slot*N + p]): rhs_p = b_p - (A * skeleton)_p.
void launch_hole_rhs_var(int dim, double* e, const double* b, const FineGeom& g, const double* coef,
                         const MeshDev& m, DevState* state, cudaStream_t s);

}  // namespace asdsm_b200
