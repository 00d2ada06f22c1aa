// Variable-coefficient operators (the reference's general ProblemSpec, fdm.hpp:18-30):
// per-point stencil coefficients sampled as fdm.cpp:63-126 does, and block-Thomas factors
// for every direct solve (slabs, coarse mesh, each hole block).
#pragma once
#include <vector>

#include "../../include/asdsm_problems.hpp"
#include "plan.hpp"

namespace asdsm_b200 {

// Per-point CSR-ordered coefficients of the operator on one tensor kind: slot s of point p at
// coef[s * npts + p]; slots = left[D-1..0], diag, right[0..D-1] (2D: 5, 3D: 7).  Entries for
// neighbours outside the kind are 0 and never used.
std::vector<double> sample_kind_coefficients(const Mesh& m, unsigned mask, const asdsm_cat::Problem& p);

// Block-Thomas factorization of one box operator (box-local x-fastest layout): blocks along
// line axis L, block size B = product of the other extents.  For block j: Dinv_j = S_j^{-1}
// (column-major B x B), l_j (coupling to block j-1), r_j (coupling to block j+1).
struct BlockThomas {
  int dim = 2;
  int ext[3] = {1, 1, 1};
  int L = 1;
  int B = 1;
  int nb = 1;
  std::vector<double> dinv;  // [box][j][k*B + i]
  std::vector<double> lo;    // [box][j][i]
  std::vector<double> up;    // [box][j][i]
};

// Factor a batch of boxes; `coef(box, local_point, slot)` returns the operator coefficient;
// couplings leaving the box are dropped (extract_block semantics, sparse.cpp:80-103).
template <typename F>
void factor_block_thomas(BlockThomas& bt, int nboxes, F coef);

BlockThomas factor_kind_box(const Mesh& m, unsigned mask, const std::vector<double>& coef, int time_axis);
BlockThomas factor_hole_boxes(const Mesh& m, const std::vector<double>& fine_coef);

}  // namespace asdsm_b200
