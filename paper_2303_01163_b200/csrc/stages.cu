// The reference's public solver stages (proj/include/asdsm/solver.hpp:70-105) as single device
// operations on a plan: richardson_extrapolate, choose_cross_points, spline_correct,
// build_skeleton (2D), merge_3d (3D) and fill_holes.  The iteration itself runs these fused
// into its own kernels; these entry points apply them to caller-given fields, with the
// reference's operation order (bitwise results for everything but fill_holes, whose direct
// solves round differently) and its argument checks.
#include <random>

#include "spline.cuh"
#include "solver.hpp"

namespace asdsm_b200 {

namespace {

// richardson_extrapolate (solver.cpp:98-109): u1 + u2 - u_cc, pointwise on the coarse mesh
__global__ void richardson_kernel(const double* __restrict__ u1, const double* __restrict__ u2,
                                  const double* __restrict__ ucc, double* __restrict__ out, i64 n) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n; i += static_cast<i64>(gridDim.x) * blockDim.x)
    out[i] = __dsub_rn(__dadd_rn(u1[i], u2[i]), ucc[i]);
}

// The coarse-mesh restriction of a field on the kind coarse along `axis` (build_projector ->
// coarse, mesh.cpp:210-260): coarse point I takes the slab point with index I_a along `axis`
// and fine index (I_b + 1) n_b - 1 along every other axis.
__global__ void restrict_to_coarse_kernel(const double* __restrict__ src, MeshDev m, int axis, double* __restrict__ out,
                                          i64 ncoarse) {
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < ncoarse;
       i += static_cast<i64>(gridDim.x) * blockDim.x) {
    i64 q = i, lin = 0, stride = 1;
    for (int b = 0; b < m.dim; ++b) {
      const int I = static_cast<int>(q % m.nc[b]);
      q /= m.nc[b];
      const int idx = b == axis ? I : (I + 1) * m.n[b] - 1;
      lin += idx * stride;
      stride *= b == axis ? m.nc[b] : m.nf[b];
    }
    out[i] = src[lin];
  }
}

// spline_correct (solver.cpp:123-150): one CTA per line J of the anisotropic mesh (coarse
// along `other`): the zero-clamped natural spline through the coarse corrections of the line,
// added at every fine point along the dense axis.
__global__ void spline_correct_kernel(const double* __restrict__ u, const double* __restrict__ ecc, MeshDev m,
                                      int dense, double* __restrict__ out) {
  extern __shared__ double sm[];
  const int nc = m.nc[dense];
  double* y = sm;             // nc + 2 knot values
  double* mm = y + nc + 2;    // second derivatives
  double* diag = mm + nc + 2;
  double* upper = diag + nc + 2;
  double* rhs = upper + nc + 2;
  const int other = 1 - dense;
  const int J = blockIdx.x;  // 0-based coarse index along `other`
  for (int c = threadIdx.x; c < nc + 2; c += blockDim.x) {
    double v = 0.0;
    if (c >= 1 && c <= nc) v = dense == 0 ? ecc[(c - 1) + static_cast<i64>(m.nc[0]) * J] : ecc[J + static_cast<i64>(m.nc[0]) * (c - 1)];
    y[c] = v;
  }
  __syncthreads();
  if (threadIdx.x == 0) spline_second_derivs(m, dense, y, mm, diag, upper, rhs);
  __syncthreads();
  const int nf = m.nf[dense];
  for (int i = threadIdx.x + 1; i <= nf; i += blockDim.x) {
    const i64 p = dense == 0 ? (i - 1) + static_cast<i64>(m.nf[0]) * J : J + static_cast<i64>(m.nc[0]) * (i - 1);
    out[p] = __dadd_rn(u[p], spline_eval(m, dense, [&](int c) { return y[c]; }, mm, i));
  }
  (void)other;
}

unsigned grid_for(i64 n) { return static_cast<unsigned>(std::min<i64>((n + 255) / 256, 4 * kNumSms)); }

}  // namespace

void Solver::stage_richardson(const double* u1, const double* u2, const double* ucc, double* out, cudaStream_t s) {
  const i64 n = g_coarse_.size;
  richardson_kernel<<<grid_for(n), 256, 0, s>>>(u1, u2, ucc, out, n);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void Solver::stage_restrict(const double* slab, int axis, double* out, cudaStream_t s) {
  const i64 n = g_coarse_.size;
  restrict_to_coarse_kernel<<<grid_for(n), 256, 0, s>>>(slab, md_, axis, out, n);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

int Solver::cross_point_choice(std::uint64_t seed) const {
  std::mt19937_64 eng(seed);  // choose_cross_points (solver.cpp:111-121)
  return static_cast<int>(eng() % 2);
}

void Solver::stage_spline_correct(const double* u, const double* ecc, int dense, double* out, cudaStream_t s) {
  if (mesh_.dim != 2) throw AsdsmError(kInvalidKind, "spline correction applies to the 2D anisotropic meshes");
  if (dense < 0 || dense > 1) throw AsdsmError(kIndexOutOfRange, "dense_axis must be 0 or 1");
  const int other = 1 - dense;
  const size_t smem = sizeof(double) * 5 * static_cast<size_t>(mesh_.nc[dense] + 2);
  spline_correct_kernel<<<static_cast<unsigned>(mesh_.nc[other]), 128, smem, s>>>(u, ecc, md_, dense, out);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void Solver::stage_skeleton(const double* const* sol, const double* u_cc, std::uint64_t seed, double* out,
                            cudaStream_t s) {
  launch_state_init(state_, 1, 1, s);
  if (coins_cap_ < 4) {
    coins_ = dev_.alloc<int>(4);
    coins_cap_ = 4;
  }
  int coins[4] = {0, 0, 0, 0};
  std::mt19937_64 eng(seed);  // choose_cross_points / merge_3d's seeded draws (solver.cpp:111-121, 309-345)
  if (mesh_.dim == 2) {
    coins[0] = static_cast<int>(eng() % 2);
  } else {
    coins[0] = static_cast<int>(eng() % 3);
    for (int i = 1; i < 4; ++i) coins[i] = static_cast<int>(eng() % 2);
  }
  ASDSM_CUDA_CHECK(cudaMemcpyAsync(coins_, coins, sizeof(coins), cudaMemcpyHostToDevice, s));
  ASDSM_CUDA_CHECK(cudaMemsetAsync(out, 0, static_cast<size_t>(g_fine_.size) * sizeof(double), s));  // holes stay 0
  if (mesh_.dim == 3) {
    skeleton(sol, u_cc, coins_, out, s);
    return;
  }
  // the general 2D skeleton kernels (the fast path's variants read the slab step's outputs)
  Skel2DArgs a{};
  a.m = md_;
  a.u_fc = sol[1];
  a.u_cf = sol[0];
  a.u_cc = u_cc;
  a.coin = coins_;
  a.e1 = cc_e1_;
  a.e2 = cc_e2_;
  a.m1 = spl_m1_;
  a.m2 = spl_m2_;
  a.out = out;
  launch_skeleton2d(a, state_, s);
}

void Solver::stage_fill(double* e, const double* b, cudaStream_t s) {
  launch_state_init(state_, 1, 1, s);
  const bool saved = ring_from_lines_;
  ring_from_lines_ = false;  // the ring comes from the caller's skeleton in e
  fill(e, b, s);
  ring_from_lines_ = saved;
}

}  // namespace asdsm_b200
