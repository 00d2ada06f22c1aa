#pragma once
#include "kernels.cuh"

namespace asdsm_b200 {

struct Merge3DArgs {
  MeshDev m;
  const double* u[3];      // slab solutions (kind coarse along a)
  const double* u_ccc;     // smooth mode coarse solution, or null
  const int* coin;         // error mode draws: [0] = slab index for u_hat, [1..3] pick_b per pair
  double* u_hat;           // triple (nc0*nc1*nc2)
  double* corr[3];         // per pair, triple
  double* mP[3];           // pair-line second derivatives: (nc_a*nc_b) x (nc_f+2)
  double* T[3];            // pair targets on the pair kinds
  double* mF1[3];          // per slab a: (nc_a*nf_f2) x (nc_f1+2)
  double* mF2[3];          // (nc_a*nf_f1) x (nc_f2+2)
  double* mF3a[3];         // (nc_a*nc_f2) x (nc_f1+2)
  double* mF3b[3];         // (nc_a*nf_f1) x (nc_f2+2)
  double* g3[3];           // (nc_a*nf_f1) x (nc_f2+2): knot values of fam3b lines
  double* corrected[3];    // corrected slabs
  double* sF1[3];          // per-interval spline coefficients (nc+1 x 4) of the fam1, fam2,
  double* sF2[3];          // fam3a and fam3b lines (spline_segments)
  double* sF3a[3];
  double* sF3b[3];
};

void launch_merge3d(const Merge3DArgs& A, double* out, DevState* st, cudaStream_t s);

}  // namespace asdsm_b200
