#pragma once
#include "kernels.cuh"

namespace asdsm_b200 {

// Both 2D slab solves of one error-mode (or smooth-mode) step in two launches.
struct Slab2DArgs {
  MeshDev m;
  int cplx;                       // mode space complex (coarse-axis cell Peclet > 2)
  // per slab a (coarse along a): eigenvectors along a, PCR tables along the fine axis
  const double* W[2];             // [k][j] (complex interleaved when cplx)
  const double* V[2];             // [j][k]
  const double* k1[2];            // [combo][level][pos]
  const double* k2[2];
  const double* invb[2];          // [combo][pos]
  int levels[2];
  const double* in_fine0;         // error mode: fine residual buffers (state selects), else null
  const double* in_fine1;
  const double* in_slab[2];       // smooth mode: assembled slab rhs
  const double* sta0;             // error mode: station copies of in_fine0 / in_fine1 (or null):
  const double* sta1;             //   [j < nc0][y] then [j < nc1][x]  (MarchArgs::sta0)
  double* modes[2];               // mode buffers [k][x] (T)
  double* sol[2];                 // slab solutions, slab layout
  int pcr_smem;                   // set by the launcher: PCR factors staged in shared memory
};

void launch_slab2d_fwd(const Slab2DArgs& A, DevState* st, cudaStream_t s);
// back transform + per-slab squared norms; the last block sets slab_norm[0..1] / have_e
// with `skel`: the last block also runs the skeleton's cross-value/spline phase (error mode)
void launch_slab2d_back(const Slab2DArgs& A, double* partials, DevState* st, double* history, bool with_norms,
                        cudaStream_t s, const Skel2DArgs* skel = nullptr);
void slab2d_prepare();

}  // namespace asdsm_b200
