#pragma once
#include "../../include/asdsm_problems.hpp"
#include "plan.hpp"

namespace asdsm_b200 {
// rhs of one tensor kind (coarse mask) in that kind's x-fastest layout (fdm.cpp:128-171).
void assemble_rhs(const Mesh& m, unsigned mask, const asdsm_cat::Problem& p, double* out);
// exact solution samples on the fine mesh.
void sample_exact(const Mesh& m, const asdsm_cat::Problem& p, double* out);
}  // namespace asdsm_b200
