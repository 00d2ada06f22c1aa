// Device side of the separable direct solver (see plan.hpp SepSolver).
#pragma once
#include "plan.hpp"

namespace asdsm_b200 {

// Solve A x = f for every box of a batch.  `in` and `out` may alias (in-place over the
// fine grid).  scratch0/scratch1 hold mode-space data: mode_size * nboxes elements of the
// mode type (double or cplx) each.
void sep_solve(const SepSolver& S, const BoxArray& in, const BoxArray& out, void* scratch0,
               void* scratch1, cudaStream_t stream);

// Back transforms only (real modes): mode-space solution in `modes` (compact layout, same
// batch as `out`) -> `out`, via `scratch` when two axes are diagonalized.
void sep_back_transform(const SepSolver& S, void* modes, const BoxArray& out, void* scratch, cudaStream_t stream);

// One-time kernel attribute setup (large dynamic shared memory for PCR); call before any
// stream capture.
void sep_prepare();

// Mode-space bytes one batch of `nboxes` needs per scratch buffer.
size_t sep_scratch_bytes(const SepSolver& S, i64 nboxes);

}  // namespace asdsm_b200
