// One-launch 2D slab step of the error-mode iteration (lines up to kPartMaxLine fine points):
// slab solves of both slabs, normalization, cross-point corrections, spline segments and the
// skeleton write, on a cluster of two CTAs (one per slab).  Replaces slab2d_fwd + slab2d_back
// (norms, fold, cc/spline) + skel2d_write_fast on the config-1 class of meshes.
#pragma once
#include "kernels.cuh"
#include "slab2d.cuh"

namespace asdsm_b200 {

struct SlabStep2DArgs {
  MeshDev m;
  const double* W[2];     // slab a: forward eigenvectors along a, [k][j]
  const double* V[2];     // [j][k]
  const double* part[2];  // SepSolver::part of slab a
  int pseg[2], pP[2], plast[2], pstride[2];
  double line_l[2], line_r[2];  // line-axis stencil coefficients of slab a
  const double* sta0;     // station copies of the residual buffers (MarchArgs::sta0/sta1)
  const double* sta1;
  double* skel_line0;     // out: u_cf / ||u_cf|| on the x-stations' lines [nc0][nf1]
  double* skel_line1;     // out: u_fc / ||u_fc|| on the y-stations' lines [nc1][nf0]
  double* corr;           // out: cross-point corrections E1 then E2 (nc0*nc1 each)
  const int* coin;        // coin[0] == 0 -> take P(u_cf) at cross points, else P(u_fc)
  double* out;            // fine array: the cross points (the rest of the skeleton: holes2d)
};

bool slabstep2d_supported(const MeshDev& m, const SepSolver* slab);
size_t slabstep2d_smem_bytes(const SlabStep2DArgs& A);
void slabstep2d_prepare();
// the cluster of this build (2 x CTAs per slab) fits on this device with A's shared memory
bool slabstep2d_launchable(const SlabStep2DArgs& A);
void launch_slabstep2d(const SlabStep2DArgs& A, DevState* st, cudaStream_t s);

}  // namespace asdsm_b200
