// Error-mode hole fill for 2D boxes (Alg. 3 / fill_core, proj/src/solver.cpp:414-432),
// specialised to the separable solver with line axis y and diagonalized axis x.
//
// In error mode the hole right-hand side is 0 - (A_ff * skeleton) on hole rows, which is
// non-zero only on the ring of points adjacent to the skeleton.  Its forward eigenvector
// transform along x is therefore analytic: for interior rows
//     fhat(k, j) = W[k][0] f(0, j) + W[k][m-1] f(m-1, j)
// and only the first/last rows need a full (O(m) per mode) transform.  One CTA per
// (hole, block of modes) builds the ring rhs from the skeleton, forms fhat on the fly and
// runs both Thomas sweeps in shared memory; the dense back transform is the DMMA GEMM.
#include "holes2d.cuh"

namespace asdsm_b200 {

namespace {

// 0 - row_dot(p, skeleton) for hole point (i, j) of the hole with fine origin (ox, oy);
// neighbours outside the box are skeleton points (or the domain boundary: no column).
__device__ __forceinline__ double ring_rhs(const double* __restrict__ e, const Hole2DArgs& A, int ox, int oy, int i,
                                           int j) {
  const Stencil& st = A.st;
  double acc = 0.0;
  const i64 Nx = A.nf0;
  if (j == 0 && oy > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[1], e[static_cast<i64>(oy - 1) * Nx + ox + i]));
  if (i == 0 && ox > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[0], e[static_cast<i64>(oy + j) * Nx + ox - 1]));
  if (i == A.m0 - 1 && ox + A.m0 < A.nf0 && st.has_right[0])
    acc = __dadd_rn(acc, __dmul_rn(st.right[0], e[static_cast<i64>(oy + j) * Nx + ox + A.m0]));
  if (j == A.m1 - 1 && oy + A.m1 < A.nf1 && st.has_right[1])
    acc = __dadd_rn(acc, __dmul_rn(st.right[1], e[static_cast<i64>(oy + A.m1) * Nx + ox + i]));
  return __dsub_rn(0.0, acc);
}

__global__ void hole2d_fwd_thomas_kernel(const double* __restrict__ e, double* __restrict__ modes, Hole2DArgs A,
                                         const DevState* state) {
  const double* __restrict__ ipiv = A.ipiv;
  const double* __restrict__ cpv = A.cp;
  if (!state->active || !state->have_e) return;
  extern __shared__ double sm[];
  const int m0 = A.m0, m1 = A.m1, KB = blockDim.x;
  double* fL = sm;
  double* fR = fL + m1;
  double* fB = fR + m1;
  double* fT = fB + m0;
  double* ys = fT + m0;  // [m1][KB] when A.y_in_smem
  const int hole = blockIdx.x;
  const int hx = hole % A.nbox0, hy = hole / A.nbox0;
  const int ox = hx * A.n0, oy = hy * A.n1;
  for (int t = threadIdx.x; t < m1; t += KB) {
    fL[t] = ring_rhs(e, A, ox, oy, 0, t);
    fR[t] = ring_rhs(e, A, ox, oy, m0 - 1, t);
  }
  for (int t = threadIdx.x; t < m0; t += KB) {
    fB[t] = ring_rhs(e, A, ox, oy, t, 0);
    fT[t] = ring_rhs(e, A, ox, oy, t, m1 - 1);
  }
  __syncthreads();
  const int k = blockIdx.y * KB + threadIdx.x;
  if (k >= m0) return;
  // full transforms of the first and last rows (8 independent loads in flight per step)
  double fb = 0.0, ft = 0.0;
  {
    int i = 0;
    for (; i + 8 <= m0; i += 8) {
      double w[8];
#pragma unroll
      for (int q = 0; q < 8; ++q) w[q] = __ldg(A.Wt + static_cast<i64>(i + q) * m0 + k);
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        fb = fma(w[q], fB[i + q], fb);
        ft = fma(w[q], fT[i + q], ft);
      }
    }
    for (; i < m0; ++i) {
      const double w = __ldg(A.Wt + static_cast<i64>(i) * m0 + k);
      fb = fma(w, fB[i], fb);
      ft = fma(w, fT[i], ft);
    }
  }
  const double w0 = __ldg(A.Wt + k), wm = __ldg(A.Wt + static_cast<i64>(m0 - 1) * m0 + k);
  const double l = A.line_left;
  double* out = modes + static_cast<i64>(hole) * m0 * m1;
  // forward sweep, pivots prefetched 8 rows ahead; y parked in smem or the mode buffer
  double y = 0.0;
  constexpr int U = 24;
  double ivn[U];
#pragma unroll
  for (int q = 0; q < U; ++q) ivn[q] = q < m1 ? __ldg(ipiv + static_cast<i64>(q) * m0 + k) : 0.0;
  for (int j0 = 0; j0 < m1; j0 += U) {
    double iv[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      iv[q] = ivn[q];
      const int jn = j0 + U + q;
      ivn[q] = jn < m1 ? __ldg(ipiv + static_cast<i64>(jn) * m0 + k) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int j = j0 + q;
      if (j >= m1) break;
      double f;
      if (j == 0) f = fb;
      else if (j == m1 - 1) f = ft;
      else f = (m0 > 1) ? fma(wm, fR[j], w0 * fL[j]) : w0 * fL[j];
      y = (j == 0) ? f * iv[q] : (f - l * y) * iv[q];
      if (A.y_in_smem) ys[j * KB + threadIdx.x] = y;
      else out[static_cast<i64>(j) * m0 + k] = y;
    }
  }
  // backward sweep, mode layout [hole][j][k]
  double x = y;
  out[static_cast<i64>(m1 - 1) * m0 + k] = x;
  double cpn[U];
#pragma unroll
  for (int q = 0; q < U; ++q) {
    const int j = m1 - 2 - q;
    cpn[q] = j >= 0 ? __ldg(cpv + static_cast<i64>(j) * m0 + k) : 0.0;
  }
  for (int j0 = m1 - 2; j0 >= 0; j0 -= U) {
    double cpj[U], yv[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      cpj[q] = cpn[q];
      const int jn = j0 - U - q;
      cpn[q] = jn >= 0 ? __ldg(cpv + static_cast<i64>(jn) * m0 + k) : 0.0;
      const int j = j0 - q;
      yv[q] = j >= 0 ? (A.y_in_smem ? ys[j * KB + threadIdx.x] : out[static_cast<i64>(j) * m0 + k]) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int j = j0 - q;
      if (j < 0) break;
      x = yv[q] - cpj[q] * x;
      out[static_cast<i64>(j) * m0 + k] = x;
    }
  }
}

// Same algorithm with every table slice this CTA needs (Wt[:, kblock], ipiv/cp[:, kblock])
// bulk-loaded into shared memory up front: one coalesced, fully overlapped load phase, then
// the transforms and both sweeps run out of shared memory (the kernel is latency bound:
// ~2 warps per SM exist in total, so memory-level parallelism has to come from the bulk load).
__global__ void hole2d_fwd_thomas_smem_kernel(const double* __restrict__ e, double* __restrict__ modes, Hole2DArgs A,
                                              const DevState* state) {
  if (!state->active || !state->have_e) return;
  extern __shared__ double sm[];
  const int m0 = A.m0, m1 = A.m1, KB = blockDim.x;
  double* fL = sm;
  double* fR = fL + m1;
  double* fB = fR + m1;
  double* fT = fB + m0;
  double* sW = fT + m0;          // [m0][KB]
  double* sI = sW + m0 * KB;     // [m1][KB]
  double* sC = sI + m1 * KB;     // [m1][KB]
  double* ys = sC + m1 * KB;     // [m1][KB]
  const int hole = blockIdx.x;
  const int hx = hole % A.nbox0, hy = hole / A.nbox0;
  const int ox = hx * A.n0, oy = hy * A.n1;
  const int kbase = blockIdx.y * KB;
  const int kcnt = min(KB, m0 - kbase);
  // stage the table slices and the skeleton neighbours of the ring with cp.async
  double* sBl = ys + m1 * KB;  // skeleton row below / above (m0 each), column left / right (m1 each)
  double* sAb = sBl + m0;
  double* sLe = sAb + m0;
  double* sRi = sLe + m1;
  for (int t = threadIdx.x; t < m0 * KB; t += KB) {
    const int i = t / KB, kk = t % KB;
    if (kk < kcnt) cp_async8(sW + t, A.Wt + static_cast<i64>(i) * m0 + kbase + kk);
    else sW[t] = 0.0;
  }
  for (int t = threadIdx.x; t < m1 * KB; t += KB) {
    const int j = t / KB, kk = t % KB;
    if (kk < kcnt) {
      cp_async8(sI + t, A.ipiv + static_cast<i64>(j) * m0 + kbase + kk);
      cp_async8(sC + t, A.cp + static_cast<i64>(j) * m0 + kbase + kk);
    }
  }
  const i64 Nx = A.nf0;
  for (int t = threadIdx.x; t < m0; t += KB) {
    if (oy > 0) cp_async8(sBl + t, e + static_cast<i64>(oy - 1) * Nx + ox + t);
    else sBl[t] = 0.0;
    if (oy + m1 < A.nf1) cp_async8(sAb + t, e + static_cast<i64>(oy + m1) * Nx + ox + t);
    else sAb[t] = 0.0;
  }
  for (int t = threadIdx.x; t < m1; t += KB) {
    if (ox > 0) cp_async8(sLe + t, e + static_cast<i64>(oy + t) * Nx + ox - 1);
    else sLe[t] = 0.0;
    if (ox + m0 < A.nf0) cp_async8(sRi + t, e + static_cast<i64>(oy + t) * Nx + ox + m0);
    else sRi[t] = 0.0;
  }
  cp_async_wait_all();
  __syncthreads();
  // ring rhs from the staged neighbours, same term order as ring_rhs (row_dot column order)
  const Stencil& st = A.st;
  auto ring = [&](int i, int j) -> double {
    double acc = 0.0;
    if (j == 0 && oy > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[1], sBl[i]));
    if (i == 0 && ox > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[0], sLe[j]));
    if (i == m0 - 1 && ox + m0 < A.nf0 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(st.right[0], sRi[j]));
    if (j == m1 - 1 && oy + m1 < A.nf1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(st.right[1], sAb[i]));
    return __dsub_rn(0.0, acc);
  };
  for (int t = threadIdx.x; t < m1; t += KB) {
    fL[t] = ring(0, t);
    fR[t] = ring(m0 - 1, t);
  }
  for (int t = threadIdx.x; t < m0; t += KB) {
    fB[t] = ring(t, 0);
    fT[t] = ring(t, m1 - 1);
  }
  __syncthreads();
  const int kk = threadIdx.x;
  const int k = kbase + kk;
  if (kk >= kcnt) return;
  double fb = 0.0, ft = 0.0;
  for (int i = 0; i < m0; ++i) {
    const double w = sW[i * KB + kk];
    fb = fma(w, fB[i], fb);
    ft = fma(w, fT[i], ft);
  }
  const double w0 = sW[kk], wm = sW[(m0 - 1) * KB + kk];
  const double l = A.line_left;
  double y = 0.0;
  for (int j = 0; j < m1; ++j) {
    double f;
    if (j == 0) f = fb;
    else if (j == m1 - 1) f = ft;
    else f = (m0 > 1) ? fma(wm, fR[j], w0 * fL[j]) : w0 * fL[j];
    const double iv = sI[j * KB + kk];
    y = (j == 0) ? f * iv : (f - l * y) * iv;
    ys[j * KB + kk] = y;
  }
  double* out = modes + static_cast<i64>(hole) * m0 * m1;
  double x = y;
  out[static_cast<i64>(m1 - 1) * m0 + k] = x;
  for (int j = m1 - 2; j >= 0; --j) {
    x = ys[j * KB + kk] - sC[j * KB + kk] * x;
    out[static_cast<i64>(j) * m0 + k] = x;
  }
}

}  // namespace

size_t hole2d_smem_bytes(int m0, int m1, int kb, bool y_in_smem, bool tables_in_smem) {
  if (tables_in_smem)
    return sizeof(double) * (4 * static_cast<size_t>(m1) + 4 * static_cast<size_t>(m0) +
                             static_cast<size_t>(m0 + 3 * m1) * kb);
  return sizeof(double) * (2 * static_cast<size_t>(m1) + 2 * static_cast<size_t>(m0) +
                           (y_in_smem ? static_cast<size_t>(m1) * kb : 0));
}

void launch_hole2d_fwd_thomas(const double* e, double* modes, const Hole2DArgs& A, DevState* state, cudaStream_t s) {
  const int kb = A.kb;
  const size_t smem = hole2d_smem_bytes(A.m0, A.m1, kb, A.y_in_smem, A.tables_in_smem);
  dim3 grid(static_cast<unsigned>(A.nbox0 * A.nbox1), static_cast<unsigned>((A.m0 + kb - 1) / kb));
  if (A.tables_in_smem) hole2d_fwd_thomas_smem_kernel<<<grid, kb, smem, s>>>(e, modes, A, state);
  else hole2d_fwd_thomas_kernel<<<grid, kb, smem, s>>>(e, modes, A, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void hole2d_prepare(size_t smem) {
  static bool done = false;
  if (done) return;
  done = true;
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole2d_fwd_thomas_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole2d_fwd_thomas_smem_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
}

}  // namespace asdsm_b200
