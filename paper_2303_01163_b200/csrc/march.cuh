#pragma once
#include "kernels.cuh"

namespace asdsm_b200 {

// kMarchCand: the residual of the update's candidate iterate (already written to the
// non-current buffer by an axpy pass) -- the 3D update runs as axpy + kMarchCand
// kMarchDotsUpdate (2D, constant coefficients): the skeleton-row step dots and the update in one
// launch -- dots, last-block step control, a grid barrier on DevState::gen, then the update
enum { kMarchResidual = 0, kMarchUpdate = 1, kMarchDots = 2, kMarchCand = 3, kMarchDotsUpdate = 4 };

struct MarchArgs {
  const double* u0;  // current iterate buffers (state->cur selects); DOTS: unused
  const double* u1;
  const double* e;   // correction (UPDATE, DOTS)
  const double* b;
  double* uo0;       // UPDATE outputs go to the non-current buffers
  double* uo1;
  double* ro0;       // residual buffers (RESIDUAL writes the current one; DOTS reads it)
  double* ro1;
  const double* r0;
  const double* r1;
  const double* exact;
  FineGeom g;
  Stencil st;
  double* partials;
  DevState* state;
  CtrlArgs ctrl;
  double* history;
  int strip;  // 2D rows per CTA (set by launch_march)
  int retry_pass;  // UPDATE: the all-rows retry of a subsampled step (runs only if state->retry)
  int sparse;      // UPDATE: sparse_residual -- hole rows get r = 0 (solver.cpp:638-643)
  int n[3];        // refinement factors (hole-row test for sparse)
  const double* coef;  // variable coefficients: coef[slot * N + p] in CSR column order, or null
  // 2D fast path: compact copies of the residual on the slab stations, one per residual
  // buffer (sta0 <-> r0, sta1 <-> r1): [j < nc0][y] (x = (j+1) n0 - 1) then [j < nc1][x]
  // (y = (j+1) n1 - 1) -- written by RESIDUAL / UPDATE so the slab gather reads them coalesced
  double* sta0;
  double* sta1;
  int nc[3];
  // DOTS on the skeleton rows only: on hole rows A e is the hole fill's own residual
  // (rounding level) -- the reference's subsampled path samples skeleton rows for that reason
  // (solver.cpp:463-465); here the full sum drops those rounding-level terms as well
  int skel_only;
  int prefetch;        // 2D persistent pass: L2-prefetch the tile this many rounds ahead (0: off)
  CtrlArgs dots_ctrl;  // kMarchDotsUpdate: the step control (kCtrlStep) between the two phases
};

// kMarchDotsUpdate needs every CTA of its grid resident at once (it waits on a grid barrier):
// true when this device's occupancy allows it (checked once)
bool dots_update_supported(const FineGeom& g);

int march_strip(const FineGeom& g);
unsigned march_blocks(const FineGeom& g);
void launch_march(int mode, const MarchArgs& A, cudaStream_t s);
// 3D constant-coefficient UPDATE / RESIDUAL as one TMA-staged z-march (stream3d.cu); opt-in
// with ASDSM_STREAM3D=1 (read at launch / capture), the register-marching passes otherwise
bool stream3d_supported(const MarchArgs& A);
void launch_stream3d(int mode, const MarchArgs& A, cudaStream_t s);

}  // namespace asdsm_b200
