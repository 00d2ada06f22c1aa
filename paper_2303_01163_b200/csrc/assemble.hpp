#pragma once
#include "../../include/asdsm_problems.hpp"
#include "plan.hpp"

namespace asdsm_b200 {
// rhs of one tensor kind (coarse mask) in that kind's x-fastest layout (fdm.cpp:128-171).
void assemble_rhs(const Mesh& m, unsigned mask, const asdsm_cat::Problem& p, double* out);
// exact solution samples on the fine mesh.
void sample_exact(const Mesh& m, const asdsm_cat::Problem& p, double* out);
// true iff alpha_a and beta_a take one value at every fine interior node (every kind's stencil
// centres are fine nodes, fdm.cpp:63-126), which is then returned in alpha[a] / beta[a]
// (spatial axes; 0 elsewhere).  Throws for a non-positive diffusion coefficient.
bool uniform_coefficients(const Mesh& m, const asdsm_cat::Problem& p, double* alpha, double* beta);
}  // namespace asdsm_b200
