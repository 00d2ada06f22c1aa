// fp64 tile GEMM on the DMMA pipe (mma.sync.m8n8k4.f64) for the eigenvector transforms:
//   out(line p, q) = sum_k in(line p, k) * M[q][k]
// over a batch of strided lines (same LineMap addressing as the scalar transform kernel).
#pragma once
#include "plan.hpp"

#include <cstdlib>

namespace asdsm_b200 {

// the even/odd kernel is used for axes of at least this many modes (below, the dense kernel's
// rounding is kept: the split's savings do not matter there)
constexpr int kEoMinModes = 64;
// (ASDSM_EO_MIN overrides; read when a transform is launched / captured)
inline int eo_min_modes() {
  const char* e = std::getenv("ASDSM_EO_MIN");
  return e ? std::atoi(e) : kEoMinModes;
}

struct GemmLines {
  int o_ext[2];
  i64 o_in[2], o_out[2];
  int nbox[3];
  i64 in_bs[3], out_bs[3];
  i64 nlines;
};

// in_es / out_es: element stride along the transform axis for input / output.
void dmma_prepare();  // kernel attributes (call before any stream capture)
// Even/odd-split transform with the half sine table of SepSolver::half (back: V, forward: W);
// half the MMAs of launch_dmma_transform.
void launch_dmma_eo_transform(bool back, const double* in, double* out, const double* half, int m, i64 in_es,
                              i64 out_es, const GemmLines& L, cudaStream_t s);
void launch_dmma_transform(const double* in, double* out, const double* M, int m, i64 in_es, i64 out_es,
                           const GemmLines& L, cudaStream_t s);
// Back transform of hole strips with the half table resident in shared memory: modes
// [box = bx + nbox0 by][k < m][j < m1] -> e[bx out_bs0 + by out_bs1 + j out_stride + i], i < m.
bool strip_back_supported(int m, int m1);
void launch_strip_back(const double* modes, double* e, const double* half, int m, int m1, int nbox0, int nbox1,
                       i64 out_bs0, i64 out_bs1, i64 out_stride, cudaStream_t s);

}  // namespace asdsm_b200
