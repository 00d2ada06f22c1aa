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
  const double w0 = __ldg(A.Wt + k);
  const double wm = m0 > 1 ? __ldg(A.Wt + static_cast<i64>(m0 - 1) * m0 + k) : 0.0;  // m0 == 1: one column
  const double l = A.line_left;
  double* out = modes + static_cast<i64>(hole) * m0 * m1 + k;  // column k of [j][k]
  // Lean sweeps: pointers advance by one row (m0) per step; pivots prefetched U rows ahead;
  // y parked in shared memory when the CTA's slice fits, else in the mode buffer.
  const double* __restrict__ ip = ipiv + k;
  const double* __restrict__ cq = cpv + k;
  double* yp = A.y_in_smem ? ys + threadIdx.x : out;
  const int ys_stride = A.y_in_smem ? KB : m0;
  constexpr int U = 16;
  double y = fb * __ldg(ip);
  yp[0] = y;
  double ivq[U];
#pragma unroll
  for (int q = 0; q < U; ++q) ivq[q] = (1 + q < m1) ? __ldg(ip + static_cast<i64>(1 + q) * m0) : 0.0;
  int j = 1;
  for (; j + U <= m1 - 1; j += U) {  // interior rows j .. j+U-1 (all < m1-1)
    double nxt[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const int jn = j + U + q;
      nxt[q] = jn < m1 ? __ldg(ip + static_cast<i64>(jn) * m0) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      const double f = fma(wm, fR[j + q], w0 * fL[j + q]);
      y = (f - l * y) * ivq[q];
      yp[static_cast<i64>(j + q) * ys_stride] = y;
    }
#pragma unroll
    for (int q = 0; q < U; ++q) ivq[q] = nxt[q];
  }
  for (int q = 0; j < m1; ++j, ++q) {  // remaining rows (the last row uses the full transform)
    const double f = (j == m1 - 1) ? ft : fma(wm, fR[j], w0 * fL[j]);
    const double iv = q < U ? ivq[q] : __ldg(ip + static_cast<i64>(j) * m0);
    y = (f - l * y) * iv;
    yp[static_cast<i64>(j) * ys_stride] = y;
  }
  // backward sweep into the mode buffer
  double x = y;
  out[static_cast<i64>(m1 - 1) * m0] = x;
  j = m1 - 2;
  for (; j - U + 1 >= 0; j -= U) {
    double cv[U], yv[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      cv[q] = __ldg(cq + static_cast<i64>(j - q) * m0);
      yv[q] = yp[static_cast<i64>(j - q) * ys_stride];
    }
#pragma unroll
    for (int q = 0; q < U; ++q) {
      x = yv[q] - cv[q] * x;
      out[static_cast<i64>(j - q) * m0] = x;
    }
  }
  for (; j >= 0; --j) {
    x = yp[static_cast<i64>(j) * ys_stride] - __ldg(cq + static_cast<i64>(j) * m0) * x;
    out[static_cast<i64>(j) * m0] = x;
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
