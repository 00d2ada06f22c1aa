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
#include "partsolve.cuh"

#include <algorithm>
#include <cstdlib>

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
#pragma unroll
  for (int q = 0; q < U; ++q) {  // remaining (<= U) rows; the last row uses the full transform
    const int jj = j + q;          // (static indices keep ivq in registers)
    if (jj < m1) {
      const double f = (jj == m1 - 1) ? ft : fma(wm, fR[jj], w0 * fL[jj]);
      y = (f - l * y) * ivq[q];
      yp[static_cast<i64>(jj) * ys_stride] = y;
    }
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

// Ring of one hole: fL, fR (columns 0 / m0-1), fB, fT (rows 0 / m1-1), ring_rhs's arithmetic
__global__ void __launch_bounds__(256) hole2d_ring_kernel(const double* __restrict__ e, Hole2DArgs A,
                                                          Hole2DPartArgs P, const DevState* state) {
  if (!state->active || !state->have_e) return;
  const int m0 = A.m0, m1 = A.m1;
  const int hole = blockIdx.x;
  const int hx = hole % A.nbox0, hy = hole / A.nbox0;
  const int ox = hx * A.n0, oy = hy * A.n1;
  double* ring = P.ring + static_cast<i64>(hole) * (2 * m1 + 2 * m0);
  for (int t = threadIdx.x; t < 2 * m1 + 2 * m0; t += blockDim.x) {
    double v;
    if (t < m1) v = ring_rhs(e, A, ox, oy, 0, t);
    else if (t < 2 * m1) v = ring_rhs(e, A, ox, oy, m0 - 1, t - m1);
    else if (t < 2 * m1 + m0) v = ring_rhs(e, A, ox, oy, t - 2 * m1, 0);
    else v = ring_rhs(e, A, ox, oy, t - 2 * m1 - m0, m1 - 1);
    ring[t] = v;
  }
}

#ifndef ASDSM_PART_HOLE_WARPS
#define ASDSM_PART_HOLE_WARPS 12  // measured 8 / 12 / 16 at config 2: 16.27 / 16.09 / 16.27 ms
#endif
constexpr int kPartHoleWarps = ASDSM_PART_HOLE_WARPS;  // mode lines (warps) per CTA

// One warp per (hole, mode k): line rhs fb, w0 fL + wm fR (interior rows), ft; partition solve;
// the line to modes[hole][k][.] (coalesced).
template <int SEG>
__global__ void __launch_bounds__(32 * kPartHoleWarps) hole2d_part_kernel(double* __restrict__ modes, Hole2DArgs A,
                                                                          Hole2DPartArgs P, const DevState* state) {
  if (!state->active || !state->have_e) return;
  extern __shared__ __align__(16) double sm[];
  const int m0 = A.m0, m1 = A.m1;
  const int lp = (m1 + 1) & ~1;  // line buffer stride
  double* fL = sm;
  double* fR = fL + m1;
  double* fB = fR + m1;
  double* fT = fB + m0;
  double* lines = fT + m0 + ((2 * m1 + 2 * m0) & 1);  // [warps][lp]
  double* tabs = lines + kPartHoleWarps * lp;         // [warps][pstride]
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int hole = blockIdx.x;
  const int k0 = blockIdx.y * kPartHoleWarps;
  const double* ring = P.ring + static_cast<i64>(hole) * (2 * m1 + 2 * m0);
  for (int t = threadIdx.x; t < 2 * m1 + 2 * m0; t += blockDim.x) cp_async8(fL + t, ring + t);
#ifdef ASDSM_PART_HOLE_STAGE
  for (int t = threadIdx.x; t < kPartHoleWarps * P.pstride; t += blockDim.x) {
    const int w = t / P.pstride, o = t - w * P.pstride;
    if (k0 + w < m0) cp_async8(tabs + t, P.part + static_cast<i64>(k0 + w) * P.pstride + o);
  }
#else
  (void)tabs;
#endif
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  const int k = k0 + warp;
  const double* Wk = P.W + static_cast<i64>(min(k, m0 - 1)) * m0;  // row k: coalesced
  const double w0 = __ldg(Wk), wm = __ldg(Wk + m0 - 1);
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  if (k >= m0) return;
  // the two full row transforms of mode k: lanes over i, then a shuffle tree
  double fb = 0.0, ft = 0.0;
  for (int i = lane; i < m0; i += 32) {
    const double w = __ldg(Wk + i);
    fb = fma(w, fB[i], fb);
    ft = fma(w, fT[i], ft);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    fb += __shfl_xor_sync(0xffffffffu, fb, o);
    ft += __shfl_xor_sync(0xffffffffu, ft, o);
  }
  double* line = lines + warp * lp;
  for (int j = lane; j < m1; j += 32)
    line[j] = j == 0 ? fb : (j == m1 - 1 ? ft : fma(wm, fR[j], w0 * fL[j]));
  __syncwarp();
#ifdef ASDSM_PART_HOLE_STAGE
  part_solve_line<SEG>(line, tabs + warp * P.pstride, m1, P.P, P.last, A.line_left, A.line_right);
#else
  // the mode's table straight from L2 (shared by every hole; loads issued ahead of the chains),
  // leaving shared memory to the lines: more CTAs per SM
  part_solve_line<SEG>(line, P.part + static_cast<i64>(k) * P.pstride, m1, P.P, P.last, A.line_left, A.line_right);
#endif
  __syncwarp();
  double* out = modes + static_cast<i64>(hole) * m0 * m1 + static_cast<i64>(k) * m1;
  for (int j = lane; j < m1; j += 32) out[j] = line[j];
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


// Whole-hole fused fill for small holes (m0, m1 <= 128): one CTA per hole runs the ring rhs,
// the analytic forward transform and the Thomas sweeps for every mode into a shared-memory
// mode tile, then the DMMA back transform (mma.sync.m8n8k4.f64) from shared memory straight
// into the hole's fine-grid positions -- no mode buffer round trip, one launch instead of two.
// Every table a phase needs (Wt, the Thomas pivots and upper factors, V) is bulk-staged into
// shared memory with cp.async before that phase, so each phase waits on one L2 round trip
// instead of one per serial step; the pivots are staged into the mode tile itself (the forward
// sweep overwrites pivot (j, k) with y(j, k) in place).
constexpr int kFusedThreads = 512;

__device__ __forceinline__ void dmma_f64(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

// rows x cols table (row stride ld in global, S in shared) -> shared, asynchronously.  Every
// CTA reads the same table at the same time: each starts at a different rotation of the
// element order so the requests spread over the L2 slices instead of queueing on one line.
__device__ __forceinline__ void stage_table(double* dst, const double* __restrict__ src, int rows, int cols, int ld,
                                            int S, int tid) {
  // (row, column) advance by the thread count without a division per element: the stride's
  // quotient and remainder once, then a carry; the rotation wraps at rows
  if ((cols & 1) == 0 && (ld & 1) == 0) {
    const int hc = cols >> 1, n = rows * hc;
    const int rot = static_cast<int>((blockIdx.x * 977u) % static_cast<unsigned>(n));
    const int dr = kFusedThreads / hc, dc = kFusedThreads - dr * hc;
    int t = tid + rot;
    if (t >= n) t -= n;
    int r = t / hc, c = t - r * hc;
    for (int t0 = tid; t0 < n; t0 += kFusedThreads) {
      cp_async16(dst + r * S + 2 * c, src + static_cast<i64>(r) * ld + 2 * c);
      r += dr;
      c += dc;
      if (c >= hc) {
        c -= hc;
        ++r;
      }
      if (r >= rows) r -= rows;
    }
  } else {
    const int n = rows * cols;
    const int rot = static_cast<int>((blockIdx.x * 977u) % static_cast<unsigned>(n));
    const int dr = kFusedThreads / cols, dc = kFusedThreads - dr * cols;
    int t = tid + rot;
    if (t >= n) t -= n;
    int r = t / cols, c = t - r * cols;
    for (int t0 = tid; t0 < n; t0 += kFusedThreads) {
      cp_async8(dst + r * S + c, src + static_cast<i64>(r) * ld + c);
      r += dr;
      c += dc;
      if (c >= cols) {
        c -= cols;
        ++r;
      }
      if (r >= rows) r -= rows;
    }
  }
}

// One warp's share of the even/odd back transform: NA j tiles (32 S apart) x NB i tiles, an
// E and an O accumulator per tile (K = kh each), the next k step's fragments loaded while the
// current step's MMAs issue.  Static counts keep the MMAs unpredicated (the caller dispatches).
template <int NA, int NB>
__device__ __forceinline__ void fused_gemm_eo(double (&ae)[4][2][2], double (&ao)[4][2][2], const double* pa,
                                              const double* pb, int kh) {
  constexpr int S = kHole2DFusedStride;
  double fe[NA], fo[NA], ge[NB], go[NB];
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    fe[a] = pa[a * 32 * S];
    fo[a] = pa[a * 32 * S + kh];
  }
#pragma unroll
  for (int b = 0; b < NB; ++b) {
    ge[b] = pb[b * 32 * S];
    go[b] = pb[b * 32 * S + kh];
  }
  for (int kk = 0; kk < kh; kk += 4) {
    const int kn = kk + 4 < kh ? kk + 4 : kk;
    double ne[NA], no[NA], me[NB], mo[NB];
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      ne[a] = pa[a * 32 * S + kn];
      no[a] = pa[a * 32 * S + kh + kn];
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      me[b] = pb[b * 32 * S + kn];
      mo[b] = pb[b * 32 * S + kh + kn];
    }
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        dmma_f64(ae[a][b], fe[a], ge[b]);
        dmma_f64(ao[a][b], fo[a], go[b]);
      }
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      fe[a] = ne[a];
      fo[a] = no[a];
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {
      ge[b] = me[b];
      go[b] = mo[b];
    }
  }
}

// Smooth-mode forward transform of a hole's rows on the DMMA pipe, in place in the mode tile:
// sY holds h+ (columns [0, kh)) and h- ([kh, 2 kh)) of every row; the modes are
// E(j, kappa) = sum_i h+(j, i) SH[i][kappa] -> column kappa (k = 2 kappa) and
// O(j, kappa) = sum_i h-(j, i) SH[i][kh + kappa] -> column kh + kappa (k = 2 kappa + 1).
// Accumulators stay in registers until every warp is done reading, then overwrite sY.
template <int NA, int NB>
__device__ __forceinline__ void fused_fwd_tiles(double (&ae)[4][2][2], double (&ao)[4][2][2], const double* pa,
                                                const double* hcol, int kh) {
  constexpr int S = kHole2DFusedStride;
  for (int kk = 0; kk < kh; kk += 4) {
    double fe[NA], fo[NA], ge[NB], go[NB];
#pragma unroll
    for (int a = 0; a < NA; ++a) {
      fe[a] = pa[a * 32 * S + kk];
      fo[a] = pa[a * 32 * S + kh + kk];
    }
#pragma unroll
    for (int b = 0; b < NB; ++b) {  // B(k = i, n = kappa) = SH[i][kappa]: column reads of the table
      ge[b] = hcol[kk * S + b * 32];
      go[b] = hcol[kk * S + kh + b * 32];
    }
#pragma unroll
    for (int a = 0; a < NA; ++a)
#pragma unroll
      for (int b = 0; b < NB; ++b) {
        dmma_f64(ae[a][b], fe[a], ge[b]);
        dmma_f64(ao[a][b], fo[a], go[b]);
      }
  }
}

__device__ __forceinline__ void fused_forward_eo(double* sY, const double* sH, int m0, int m1, int kh, int mh,
                                                 int tid) {
  constexpr int S = kHole2DFusedStride;
  const int lane = tid & 31, warp = tid >> 5;
  const int jg = warp >> 2, ig = (warp + jg) & 3;
  const int JP = (m1 + 7) & ~7;
  const int jt = JP >> 3, it = (kh + 7) >> 3;
  double ae[4][2][2], ao[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) ae[a][b][0] = ae[a][b][1] = ao[a][b][0] = ao[a][b][1] = 0.0;
  const int r8 = lane >> 2, c4 = lane & 3;
  const double* pa = sY + (jg * 8 + r8) * S + c4;
  const double* hcol = sH + c4 * S + ig * 8 + r8;  // + kk * S (k = i row) + tile * 32 (n = kappa)
  const int na = min(4, max(0, (jt - jg + 3) >> 2));
  const int nb = min(2, max(0, (it - ig + 3) >> 2));
  switch (na * 3 + nb) {
#define ASDSM_FWD_CASE(NA, NB) \
  case NA * 3 + NB:            \
    fused_fwd_tiles<NA, NB>(ae, ao, pa, hcol, kh); \
    break;
    ASDSM_FWD_CASE(1, 1) ASDSM_FWD_CASE(1, 2) ASDSM_FWD_CASE(2, 1) ASDSM_FWD_CASE(2, 2)
    ASDSM_FWD_CASE(3, 1) ASDSM_FWD_CASE(3, 2) ASDSM_FWD_CASE(4, 1) ASDSM_FWD_CASE(4, 2)
#undef ASDSM_FWD_CASE
    default:
      break;
  }
  __syncthreads();  // every warp has read its h tiles
  const int me = (m0 + 1) >> 1, mo = m0 >> 1;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int j = (jg + 4 * a) * 8 + r8;
    if (a >= na || j >= m1) continue;
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      if (b >= nb) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kap = (ig + 4 * b) * 8 + 2 * c4 + h;
        if (kap < me) sY[j * S + kap] = ae[a][b][h];
        if (kap < mo) sY[j * S + kh + kap] = ao[a][b][h];
      }
    }
  }
  (void)mh;
}

// Error-mode hole fill, one CTA per hole (holes up to 108 x 128):
//   P0  pivots -> shared (cp.async) ; ring rhs from the skeleton
//   P1  full forward transforms of the first / last ring rows, W = c S D^-1 applied through
//       the even/odd half sine table (W never leaves L2)
//   P2  twisted Thomas per mode (top/bottom threads meet in the middle), modes x into shared
//       memory with even/odd-permuted columns
//   P4  half sine table -> shared over the dead pivots
//   P5  back transform on the DMMA pipe, even/odd split: E = X_even S_e^T, O = X_odd S_o^T
//       over ceil(m0/2) rows -- half the MMAs of a dense V, and out(i) = sc_i (E + O),
//       out(m0-1-i) = sc_{m0-1-i} (E - O) written straight into the fine array
template <bool SMOOTH>
__global__ void __launch_bounds__(kFusedThreads, 1)
    hole2d_fused_kernel(double* __restrict__ e, Hole2DArgs A, const double* __restrict__ bvec, const DevState* state) {
  pdl_launch_dependents();
#ifdef ASDSM_FUSED_TRACE  // per-phase clock64 stamps of CTAs 0 and 55, printed at the end
  long long T[8] = {clock64(), 0, 0, 0, 0, 0, 0, 0};
#define FUSED_STAMP(i) T[i] = clock64()
#else
#define FUSED_STAMP(i)
#endif
  constexpr int S = kHole2DFusedStride;  // compile-time row stride: every row offset is an immediate
  extern __shared__ __align__(16) double sm[];
  const int m0 = A.m0, m1 = A.m1;
  const int kh = half_sine_kh(m0), hr = half_sine_rows(m0);
  const int mh = (m0 + 1) >> 1;  // rows of the half transform
  const int JP = (m1 + 7) & ~7;
  const int NP = m1 - ((m1 - 1) >> 1);  // pivot rows the twisted sweeps use (distance < NP)
  const double* __restrict__ SH = A.half;               // [hr][2 kh]
  const double* __restrict__ sc = A.half + hr * 2 * kh; // scale_i
  const double* __restrict__ ci = sc + m0;              // (2/(m0+1)) / scale_i
  double* sY = sm;            // [JP][S]: sweep values y / z, then the modes x (row j, permuted col)
  double* sH = sY + JP * S;   // [hr][S]: half sine table (resident for P1 and P5)
  double* sP = sH + hr * S;   // [NP][S]: Thomas pivots (row t = distance from the own end, mode k)
  double* fL = sP + NP * S;
  double* fR = fL + m1;
  double* fB = fR + m1;
  double* fT = fB + m0;
  double* part = fT + m0;     // [4][2][128] partial sums of the full row transforms
  double* xch = part + 1024;  // [2 sides][2][128] values exchanged at the meeting rows
  double* scs = xch + 512;    // [m0] scale_i
  double* hv = scs + 128;     // [4][64] ring-row pair sums h+ / h- of fB and fT (P0: [4][128] ring sides)
  const int tid = threadIdx.x;
  const int hole = blockIdx.x;
  const int hx = hole % A.nbox0, hy = hole / A.nbox0;
  const int ox = hx * A.n0, oy = hy * A.n1;
  // P0 (the tables are constant: staged while the previous kernel drains)
  stage_table(sP, A.ipiv, NP, m0, m0, S, tid);
  stage_table(sH, SH, hr, 2 * kh, 2 * kh, S, tid);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  pdl_wait();
  if (!state->active || !state->have_e) {
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    return;
  }
  auto zero_kpad = [&]() {  // zero the k padding of the mode tile (even / odd mode counts me / mo)
    const int me = (m0 + 1) >> 1, mo = m0 >> 1;
    const int pe = kh - me, po = kh - mo;
    for (int t = tid; t < JP * (pe + po); t += kFusedThreads) {
      const int r = t / (pe + po), c = t % (pe + po);
      sY[r * S + (c < pe ? me + c : kh + mo + (c - pe))] = 0.0;
    }
  };
  if (!SMOOTH) zero_kpad();
  if (tid >= 128 && tid - 128 < m0) scs[tid - 128] = __ldg(sc + tid - 128);
  const i64 Nxg = A.nf0;
  if (SMOOTH) {
    // smooth mode: rhs = b - A_hs skeleton on every hole row (hole_rhs_kernel's arithmetic),
    // pre-scaled by c D^-1 for the forward transform: g(j, i) in natural columns
    for (int t = tid; t < m1 * m0; t += kFusedThreads) {
      const int j = t / m0, i = t - j * m0;
      double f = __ldg(bvec + static_cast<i64>(oy + j) * Nxg + ox + i);
      if (i == 0 || i == m0 - 1 || j == 0 || j == m1 - 1) f = __dadd_rn(f, ring_rhs(e, A, ox, oy, i, j));
      sY[j * S + i] = f * __ldg(ci + i);
    }
  } else if (A.skel_line0 != nullptr) {
    // the four skeleton sides of this hole: line value / norm + sum_k B[pos][k] E[k] (the same
    // arithmetic the skeleton write used), into the ring arrays' spare room (hv: 4 x 128)
    double* sB = hv;        // bottom row (y-station hy-1), x = ox + i
    double* sT = hv + 128;  // top row (y-station hy)
    double* sL = hv + 256;  // left column (x-station hx-1), y = oy + j
    double* sR = hv + 384;  // right column (x-station hx)
    const int nc0 = A.nc0, nc1 = A.nc1, ncc = nc0 * nc1;
    const double* E1 = A.corr;
    const double* E2 = A.corr + ncc;
    for (int t = tid; t < 2 * m0 + 2 * m1; t += kFusedThreads) {
      int side, q;
      if (t < m0) { side = 0; q = t; }
      else if (t < 2 * m0) { side = 1; q = t - m0; }
      else if (t < 2 * m0 + m1) { side = 2; q = t - 2 * m0; }
      else { side = 3; q = t - 2 * m0 - m1; }
      // row sides: station J = hy - 1 / hy at x = ox + q, basis of axis 0, E1 row J;
      // column sides: station I = hx - 1 / hx at y = oy + q, basis of axis 1, E2 column I
      const bool row = side < 2;
      const int stn = row ? hy - 1 + side : hx - 1 + (side - 2);
      const int nk = row ? nc0 : nc1;
      const int pos = row ? ox + q : oy + q;
      double v = 0.0;
      if (stn >= 0 && stn < (row ? nc1 : nc0)) {
        const double* bb = (row ? A.basis0 : A.basis1) + static_cast<i64>(pos) * nk;
        const double* ee = row ? E1 + nc0 * stn : E2 + stn;
        const int es = row ? 1 : nc0;
        const double lv = __ldg((row ? A.skel_line1 + static_cast<i64>(stn) * A.nf0 : A.skel_line0 + static_cast<i64>(stn) * A.nf1) + pos);
        constexpr int kU = 12;  // every load of the dot product in flight at once
        double bq[kU], eq[kU];
#pragma unroll
        for (int k = 0; k < kU; ++k) {
          bq[k] = k < nk ? __ldg(bb + k) : 0.0;
          eq[k] = k < nk ? __ldg(ee + k * es) : 0.0;
        }
        double sp = 0.0;
#pragma unroll
        for (int k = 0; k < kU; ++k)
          if (k < nk) sp = fma(bq[k], eq[k], sp);
        for (int k = kU; k < nk; ++k) sp = fma(__ldg(bb + k), __ldg(ee + k * es), sp);
        v = __dadd_rn(lv, sp);
        if (side == 0) e[static_cast<i64>(oy - 1) * Nxg + pos] = v;  // owned: the bottom row
        if (side == 2) e[static_cast<i64>(pos) * Nxg + ox - 1] = v;  // owned: the left column
      }
      (side == 0 ? sB : side == 1 ? sT : side == 2 ? sL : sR)[q] = v;
    }
    __syncthreads();
    const Stencil& st = A.st;
    auto ring = [&](int i, int j) -> double {  // ring_rhs's terms and order on the computed sides
      double acc = 0.0;
      if (j == 0 && oy > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[1], sB[i]));
      if (i == 0 && ox > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[0], sL[j]));
      if (i == m0 - 1 && ox + m0 < A.nf0 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(st.right[0], sR[j]));
      if (j == m1 - 1 && oy + m1 < A.nf1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(st.right[1], sT[i]));
      return __dsub_rn(0.0, acc);
    };
    double rl = 0.0, rr = 0.0, rb = 0.0, rt = 0.0;  // read before the arrays are overwritten
    if (tid < m1) {
      rl = ring(0, tid);
      rr = ring(m0 - 1, tid);
    } else if (tid >= 256 && tid - 256 < m0) {
      rb = ring(tid - 256, 0);
      rt = ring(tid - 256, m1 - 1);
    }
    __syncthreads();
    if (tid < m1) {
      fL[tid] = rl;
      fR[tid] = rr;
    } else if (tid >= 256 && tid - 256 < m0) {
      const double c = __ldg(ci + tid - 256);
      fB[tid - 256] = rb * c;
      fT[tid - 256] = rt * c;
    }
  } else if (tid < m1) {
    fL[tid] = ring_rhs(e, A, ox, oy, 0, tid);
    fR[tid] = ring_rhs(e, A, ox, oy, m0 - 1, tid);
  } else if (tid >= 256 && tid - 256 < m0) {
    const int i = tid - 256;
    const double c = __ldg(ci + i);  // the ring rows enter W through D^-1: pre-scale
    fB[i] = ring_rhs(e, A, ox, oy, i, 0) * c;
    fT[i] = ring_rhs(e, A, ox, oy, i, m1 - 1) * c;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  FUSED_STAMP(1);
  // P1: fb[k] = sum_{i<mh} s_ik (g_i +- g_{m0-1-i}) (sign (-1)^k), g = c D^-1 f; i in four groups
  const int side = tid >> 7, k = tid & 127;  // sweeps: warps 0-3 top side, warps 4-7 bottom side
  const bool sweeper = side < 2 && k < m0;
  const int colk = (k & 1) ? kh + (k >> 1) : (k >> 1);
  double w0 = 0.0, wm = 0.0;
  if (SMOOTH) {
    // h+ / h- of every row into columns [0, kh) / [kh, 2 kh) in place (values read before the
    // barrier, written after), K padding zeroed; then modes = h S^T on the DMMA pipe
    constexpr int kPer = 14;  // >= ceil(128 * 54 / 512)
    double hp[kPer], hm[kPer];
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int t = tid + u * kFusedThreads, j = t / kh, i = t - j * kh;
      hp[u] = hm[u] = 0.0;
      if (j < m1 && i < mh) {
        const double gi = sY[j * S + i], gm = sY[j * S + m0 - 1 - i];
        const bool mid = (m0 - 1 - i) == i;
        hp[u] = mid ? gi : gi + gm;
        hm[u] = mid ? gi : gi - gm;
      }
    }
    __syncthreads();
#pragma unroll
    for (int u = 0; u < kPer; ++u) {
      const int t = tid + u * kFusedThreads, j = t / kh, i = t - j * kh;
      if (j < JP) {
        sY[j * S + i] = hp[u];
        sY[j * S + kh + i] = hm[u];
      }
    }
    __syncthreads();
    fused_forward_eo(sY, sH, m0, m1, kh, mh, tid);
    zero_kpad();
  } else if (tid < mh) {  // pair sums of the pre-scaled ring rows: h+ (even k) and h- (odd k)
    const int i = tid, im = m0 - 1 - tid;
    hv[i] = im == i ? fB[i] : fB[i] + fB[im];
    hv[64 + i] = im == i ? fB[i] : fB[i] - fB[im];
    hv[128 + i] = im == i ? fT[i] : fT[i] + fT[im];
    hv[192 + i] = im == i ? fT[i] : fT[i] - fT[im];
  }
  __syncthreads();
  if (!SMOOTH && k < m0) {
    const int g = tid >> 7;
    const int q = (mh + 3) >> 2;
    const int i0 = g * q, i1 = min(mh, i0 + q);
    const bool odd = k & 1;
    const double* hb = hv + (odd ? 64 : 0);
    const double* ht = hv + (odd ? 192 : 128);
    double pb = 0.0, pt = 0.0;
#pragma unroll 4
    for (int i = i0; i < i1; ++i) {
      const double s = sH[i * S + colk];
      pb = fma(s, hb[i], pb);
      pt = fma(s, ht[i], pt);
    }
    part[(2 * g) * 128 + k] = pb;
    part[(2 * g + 1) * 128 + k] = pt;
    if (sweeper) {
      const double s0 = sH[colk];
      w0 = s0 * __ldg(ci);
      wm = (odd ? -s0 : s0) * __ldg(ci + m0 - 1);
    }
  }
  __syncthreads();
  FUSED_STAMP(2);
  // P2: twisted (two-sided) Thomas per mode: the top thread eliminates rows 0..p downward, the
  // bottom thread rows m1-1..p+1 upward (the bottom-up pivots of a Toeplitz tridiagonal are the
  // top-down ones by distance from the end), they meet in a 2x2 solve and substitute outward --
  // chains half as long as one Thomas sweep.  Upper factors are r * pivot (top) / l * pivot.
  const double l = A.line_left, rr = A.line_right;
  const int p = (m1 - 1) >> 1;
  const int n1 = side ? m1 - 1 - p : p + 1;  // rows this side eliminates
  const double* pv = sP + k;                 // pivot t of this mode: pv[t * S]
  if (sweeper) {
    // error mode: the mode-space rhs of interior rows is w0 fL + wm fR (ring-only rhs), the two
    // boundary rows the full transforms fb / ft; smooth mode: read from the mode tile
    const double fb = SMOOTH ? 0.0 : ((part[k] + part[256 + k]) + part[512 + k]) + part[768 + k];
    const double ft = SMOOTH ? 0.0 : ((part[128 + k] + part[384 + k]) + part[640 + k]) + part[896 + k];
    const double cf = side ? rr : l, cb = side ? l : rr;
    double y;
    if (side == 0) {  // rows 0 .. p
      double* yv = sY + colk;
      y = (SMOOTH ? yv[0] : fb) * pv[0];
      yv[0] = y;
      int t = 1;
      for (; t + 8 <= n1; t += 8) {
        double pq[8], fq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          pq[q] = pv[(t + q) * S];
          fq[q] = SMOOTH ? yv[(t + q) * S] : fma(wm, fR[t + q], w0 * fL[t + q]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          y = (fq[q] - cf * y) * pq[q];
          yv[(t + q) * S] = y;
        }
      }
      for (; t < n1; ++t) {
        y = ((SMOOTH ? yv[t * S] : fma(wm, fR[t], w0 * fL[t])) - cf * y) * pv[t * S];
        yv[t * S] = y;
      }
    } else {  // rows m1-1 .. p+1
      double* yv = sY + (m1 - 1) * S + colk;  // row m1-1-t at yv[-t * S]
      const double* fl = fL + (m1 - 1);
      const double* fr = fR + (m1 - 1);
      y = (SMOOTH ? yv[0] : ft) * pv[0];
      yv[0] = y;
      int t = 1;
      for (; t + 8 <= n1; t += 8) {
        double pq[8], fq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          pq[q] = pv[(t + q) * S];
          fq[q] = SMOOTH ? yv[-(t + q) * S] : fma(wm, fr[-(t + q)], w0 * fl[-(t + q)]);
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          y = (fq[q] - cf * y) * pq[q];
          yv[-(t + q) * S] = y;
        }
      }
      for (; t < n1; ++t) {
        y = ((SMOOTH ? yv[-t * S] : fma(wm, fr[-t], w0 * fl[-t])) - cf * y) * pv[t * S];
        yv[-t * S] = y;
      }
    }
    xch[(2 * side) * 128 + k] = y;
    xch[(2 * side + 1) * 128 + k] = cb * pv[(n1 - 1) * S];
  }
  FUSED_STAMP(3);
  __syncthreads();
  if (sweeper) {
    const double yp = xch[k], cpp = xch[128 + k];       // top: y_p, c'_p
    const double zq = xch[256 + k], aq = xch[384 + k];  // bottom: z_{p+1}, a'_{p+1}
    const double xp = (yp - cpp * zq) / (1.0 - cpp * aq);
    const double xq = zq - aq * xp;
    FUSED_STAMP(4);
    const double cb = side ? l : rr;
    // substitute back toward the own end: x_t = y_t - cb * piv_t * x_{t+1}
    double x = side ? xq : xp;
    int t = n1 - 2;
    if (side == 0) {
      double* yv = sY + colk;
      yv[(n1 - 1) * S] = x;
      for (; t - 7 >= 0; t -= 8) {
        double yq[8], cq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          yq[q] = yv[(t - q) * S];
          cq[q] = cb * pv[(t - q) * S];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          x = yq[q] - cq[q] * x;
          yv[(t - q) * S] = x;
        }
      }
      for (; t >= 0; --t) {
        x = yv[t * S] - (cb * pv[t * S]) * x;
        yv[t * S] = x;
      }
    } else {
      double* yv = sY + (m1 - 1) * S + colk;
      yv[-(n1 - 1) * S] = x;
      for (; t - 7 >= 0; t -= 8) {
        double yq[8], cq[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          yq[q] = yv[-(t - q) * S];
          cq[q] = cb * pv[(t - q) * S];
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          x = yq[q] - cq[q] * x;
          yv[-(t - q) * S] = x;
        }
      }
      for (; t >= 0; --t) {
        x = yv[-t * S] - (cb * pv[t * S]) * x;
        yv[-t * S] = x;
      }
    }
  }
  FUSED_STAMP(6);
  __syncthreads();
  __syncthreads();
  FUSED_STAMP(7);
  // P5: 16 warps; warp w takes j tiles jg + 4a and half-row tiles ig + 4b with jg = w / 4,
  // ig = (w + jg) % 4, so each SM sub-partition (w % 4) holds one warp of every (jg, ig)
  // diagonal and the DMMA work is balanced across the four pipes.
  const int lane = tid & 31, warp = tid >> 5;
  const int jg = warp >> 2, ig = (warp + jg) & 3;
  const int jt = JP >> 3, it = hr >> 3;
  double ae[4][2][2], ao[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) ae[a][b][0] = ae[a][b][1] = ao[a][b][0] = ao[a][b][1] = 0.0;
  const int r8 = lane >> 2, c4 = lane & 3;
  const double* pa = sY + (jg * 8 + r8) * S + c4;
  const double* pb = sH + (ig * 8 + r8) * S + c4;
  const int na = min(4, max(0, (jt - jg + 3) >> 2));
  const int nb = min(2, max(0, (it - ig + 3) >> 2));
  switch (na * 3 + nb) {
#define ASDSM_FUSED_CASE(NA, NB) \
  case NA * 3 + NB:              \
    fused_gemm_eo<NA, NB>(ae, ao, pa, pb, kh); \
    break;
    ASDSM_FUSED_CASE(1, 1) ASDSM_FUSED_CASE(1, 2) ASDSM_FUSED_CASE(2, 1) ASDSM_FUSED_CASE(2, 2)
    ASDSM_FUSED_CASE(3, 1) ASDSM_FUSED_CASE(3, 2) ASDSM_FUSED_CASE(4, 1) ASDSM_FUSED_CASE(4, 2)
#undef ASDSM_FUSED_CASE
    default:
      break;
  }
  FUSED_STAMP(5);
  // epilogue: each lane holds E, O at rows (j, i), (j, i+1) of its tiles: out(i) = sc_i (E+O)
  // and the mirror out(m0-1-i) = sc (E-O), stored as pairs (16-byte stores where aligned)
  const i64 Nx = A.nf0;
#pragma unroll
  for (int a = 0; a < 4; ++a) {
    const int j = (jg + 4 * a) * 8 + r8;
    if (a >= na || j >= m1) continue;
    double* row = e + static_cast<i64>(oy + j) * Nx + ox;
    const bool al = ((reinterpret_cast<uintptr_t>(row) & 15) == 0);
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      if (b >= nb) continue;
      const int i = (ig + 4 * b) * 8 + 2 * c4;  // i even
      if (i >= mh) continue;
      const int im = m0 - 1 - i;
      const double E0 = ae[a][b][0], O0 = ao[a][b][0], E1 = ae[a][b][1], O1 = ao[a][b][1];
      const double lo0 = scs[i] * (E0 + O0), hi0 = scs[im] * (E0 - O0);
      if (i + 1 < mh) {
        const double lo1 = scs[i + 1] * (E1 + O1), hi1 = scs[im - 1] * (E1 - O1);
        if (al) *reinterpret_cast<double2*>(row + i) = make_double2(lo0, lo1);
        else {
          row[i] = lo0;
          row[i + 1] = lo1;
        }
        if (im - 1 > i + 1) {  // mirrors distinct from the direct pair
          if (al && ((im - 1) & 1) == 0) *reinterpret_cast<double2*>(row + im - 1) = make_double2(hi1, hi0);
          else {
            row[im - 1] = hi1;
            row[im] = hi0;
          }
        }
      } else {
        row[i] = lo0;
        if (im != i) row[im] = hi0;
      }
    }
  }
#ifdef ASDSM_FUSED_TRACE
  {
    __syncthreads();
    const long long T8 = clock64();
    if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == 55))
      printf("FUSEDDBG blk %d stage+ring %lld rowtf %lld elim %lld div %lld subst %lld gemm %lld epi %lld\n",
             blockIdx.x, T[1] - T[0], T[2] - T[1], T[3] - T[2], T[4] - T[3], T[6] - T[4], T[5] - T[7], T8 - T[5]);
  }
#endif
#undef FUSED_STAMP
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

size_t hole2d_fused_smem_bytes(int m0, int m1) {
  const size_t S = kHole2DFusedStride;
  const size_t jp = (m1 + 7) & ~7;
  const size_t np = m1 - ((m1 - 1) >> 1);
  return sizeof(double) * ((jp + half_sine_rows(m0) + np) * S + 2 * static_cast<size_t>(m0 + m1) + 17 * 128);
}

bool hole2d_fused_fits(int m0, int m1) {
  return m0 >= 2 && m1 >= 2 && m0 <= 128 && m1 <= 128 && 2 * half_sine_kh(m0) <= kHole2DFusedStride &&
         hole2d_fused_smem_bytes(m0, m1) <= kHole2DFusedMaxSmem;
}

void launch_hole2d_fused(double* e, const Hole2DArgs& A, const double* b, DevState* state, cudaStream_t s) {
  const size_t smem = hole2d_fused_smem_bytes(A.m0, A.m1);
  const unsigned grid = static_cast<unsigned>(A.nbox0 * A.nbox1);
  if (b) launch_pdl(hole2d_fused_kernel<true>, grid, kFusedThreads, smem, s, e, A, b, static_cast<const DevState*>(state));
  else launch_pdl(hole2d_fused_kernel<false>, grid, kFusedThreads, smem, s, e, A, static_cast<const double*>(nullptr),
                  static_cast<const DevState*>(state));
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

bool hole2d_part_supported(int seg) { return seg == 4 || seg == 8 || seg == 12 || seg == 16; }

namespace {
constexpr int kSepRowsJ = 64;     // rows j per CTA (coalesced)
// k groups per CTA (each thread sums every KG-th mode): 8, or 4 with more than 4 separators
__host__ __device__ constexpr int sep_rows_kg(int ns) { return ns <= 4 ? 8 : 4; }

// One CTA per (hole, 64 rows j), 8 k-groups: thread (jj, g) sums the modes k = g, g + 8, ... of
// row j for the NS separators (loads of consecutive k in flight together), then the k-groups
// combine in shared memory in a fixed order.
template <int NS, int kSepRowsKG = sep_rows_kg(NS)>
__global__ void __launch_bounds__(kSepRowsJ * kSepRowsKG) hole2d_sep_rows_kernel(const double* __restrict__ modes,
                                                                                const double* __restrict__ V,
                                                                                double* __restrict__ e, Hole2DArgs A,
                                                                                const DevState* state,
                                                                                double* __restrict__ dense) {
  if (!state->active || !state->have_e) return;
  extern __shared__ double vs[];  // [s][k]: rows i_s of V, then the k-group partials [g][s][jj]
  const int m0 = A.m0, m1 = A.m1, w1 = (m0 + 1) / (NS + 1);
  for (int t = threadIdx.x; t < NS * m0; t += blockDim.x) {
    const int sidx = t / m0, k = t - sidx * m0;
    vs[t] = __ldg(V + static_cast<i64>((sidx + 1) * w1 - 1) * m0 + k);
  }
  __syncthreads();
  double* part = vs + NS * m0;
  const int hole = blockIdx.x;
  const int jj = threadIdx.x % kSepRowsJ, g = threadIdx.x / kSepRowsJ;
  const int j = blockIdx.y * kSepRowsJ + jj;
  double acc[NS];
#pragma unroll
  for (int q = 0; q < NS; ++q) acc[q] = 0.0;
  if (j < m1) {
    const double* md = modes + static_cast<i64>(hole) * m0 * m1 + j;
    int k = g;
    for (; k + 3 * kSepRowsKG < m0; k += 4 * kSepRowsKG) {
      double w[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) w[u] = __ldg(md + static_cast<i64>(k + u * kSepRowsKG) * m1);
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int q = 0; q < NS; ++q) acc[q] = fma(vs[q * m0 + k + u * kSepRowsKG], w[u], acc[q]);
    }
    for (; k < m0; k += kSepRowsKG) {
      const double w = __ldg(md + static_cast<i64>(k) * m1);
#pragma unroll
      for (int q = 0; q < NS; ++q) acc[q] = fma(vs[q * m0 + k], w, acc[q]);
    }
  }
#pragma unroll
  for (int q = 0; q < NS; ++q) part[(g * NS + q) * kSepRowsJ + jj] = acc[q];
  __syncthreads();
  if (g != 0 || j >= m1) return;
  const int hx = hole % A.nbox0, hy = hole / A.nbox0;
  double* out = e + static_cast<i64>(hy * A.n1 + j) * A.nf0 + hx * A.n0;
#pragma unroll
  for (int q = 0; q < NS; ++q) {
    double v = 0.0;
#pragma unroll
    for (int gg = 0; gg < kSepRowsKG; ++gg) v += part[(gg * NS + q) * kSepRowsJ + jj];
    if (dense) dense[(static_cast<i64>(hole) * NS + q) * m1 + j] = v;  // [hole][s][j]
    else out[(q + 1) * w1 - 1] = v;
  }
}

// Separator values [s][j] (one column per hole, from the separator GEMM) into the fine array.
__global__ void hole2d_sep_scatter_kernel(const double* __restrict__ sep, double* __restrict__ e, Hole2DArgs A,
                                          int p, const DevState* state) {
  if (!state->active || !state->have_e) return;
  const int m1 = A.m1, ns = p - 1, w1 = (A.m0 + 1) / p;
  const int hole = blockIdx.x;
  const int hx = hole % A.nbox0, hy = hole / A.nbox0;
  const double* src = sep + static_cast<i64>(hole) * ns * m1;
  for (int t = threadIdx.x; t < ns * m1; t += blockDim.x) {
    const int q = t / m1, j = t - q * m1;
    e[static_cast<i64>(hy * A.n1 + j) * A.nf0 + hx * A.n0 + (q + 1) * w1 - 1] = src[t];
  }
}
}  // namespace

void launch_hole2d_sep_scatter(const double* sep, double* e, const Hole2DArgs& A, int p, DevState* state,
                               cudaStream_t s) {
  hole2d_sep_scatter_kernel<<<static_cast<unsigned>(A.nbox0 * A.nbox1), 256, 0, s>>>(sep, e, A, p, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_hole2d_sep_rows(const double* modes, const double* V, double* e, const Hole2DArgs& A, int p,
                            DevState* state, cudaStream_t s, double* dense) {
  if (p < 2 || p > 10 || (A.m0 + 1) % p != 0) throw AsdsmError(kUnsupported, "hole strip split");
  const dim3 grid(static_cast<unsigned>(A.nbox0 * A.nbox1), static_cast<unsigned>((A.m1 + kSepRowsJ - 1) / kSepRowsJ));
  const size_t smem = sizeof(double) * static_cast<size_t>(p - 1) * (A.m0 + sep_rows_kg(p - 1) * kSepRowsJ);
  if (smem > 48 * 1024) throw AsdsmError(kUnsupported, "hole strip split: separator table exceeds shared memory");
  const unsigned nt = kSepRowsJ * sep_rows_kg(p - 1);
  switch (p - 1) {
    case 1: hole2d_sep_rows_kernel<1><<<grid, nt, smem, s>>>(modes, V, e, A, state, dense); break;
    case 2: hole2d_sep_rows_kernel<2><<<grid, nt, smem, s>>>(modes, V, e, A, state, dense); break;
    case 3: hole2d_sep_rows_kernel<3><<<grid, nt, smem, s>>>(modes, V, e, A, state, dense); break;
    case 4: hole2d_sep_rows_kernel<4><<<grid, nt, smem, s>>>(modes, V, e, A, state, dense); break;
    case 5: hole2d_sep_rows_kernel<5><<<grid, nt, smem, s>>>(modes, V, e, A, state, dense); break;
    case 6: hole2d_sep_rows_kernel<6><<<grid, nt, smem, s>>>(modes, V, e, A, state, dense); break;
    case 7: hole2d_sep_rows_kernel<7><<<grid, nt, smem, s>>>(modes, V, e, A, state, dense); break;
    case 8: hole2d_sep_rows_kernel<8><<<grid, nt, smem, s>>>(modes, V, e, A, state, dense); break;
    default: hole2d_sep_rows_kernel<9><<<grid, nt, smem, s>>>(modes, V, e, A, state, dense); break;
  }
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_hole2d_ring(const double* e, const Hole2DArgs& A, const Hole2DPartArgs& P, DevState* state,
                        cudaStream_t s) {
  hole2d_ring_kernel<<<static_cast<unsigned>(A.nbox0 * A.nbox1), 256, 0, s>>>(e, A, P, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_hole2d_part(double* modes, const Hole2DArgs& A, const Hole2DPartArgs& P, DevState* state, cudaStream_t s) {
  const int lp = (A.m1 + 1) & ~1;
#ifdef ASDSM_PART_HOLE_STAGE
  const size_t tab = kPartHoleWarps * static_cast<size_t>(P.pstride);
#else
  const size_t tab = 0;
#endif
  const size_t smem = sizeof(double) * (2 * static_cast<size_t>(A.m1 + A.m0) + 1 + kPartHoleWarps * static_cast<size_t>(lp) + tab);
  if (smem > 100 * 1024) throw AsdsmError(kUnsupported, "partitioned hole solve exceeds shared memory");
  const dim3 grid(static_cast<unsigned>(A.nbox0 * A.nbox1), static_cast<unsigned>((A.m0 + kPartHoleWarps - 1) / kPartHoleWarps));
  switch (P.seg) {
    case 4: hole2d_part_kernel<4><<<grid, 32 * kPartHoleWarps, smem, s>>>(modes, A, P, state); break;
    case 8: hole2d_part_kernel<8><<<grid, 32 * kPartHoleWarps, smem, s>>>(modes, A, P, state); break;
    case 12: hole2d_part_kernel<12><<<grid, 32 * kPartHoleWarps, smem, s>>>(modes, A, P, state); break;
    case 16: hole2d_part_kernel<16><<<grid, 32 * kPartHoleWarps, smem, s>>>(modes, A, P, state); break;
    default: throw AsdsmError(kUnsupported, "partitioned hole solve: segment length");
  }
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
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole2d_fused_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kHole2DFusedMaxSmem)));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole2d_part_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole2d_part_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole2d_part_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole2d_part_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 100 * 1024));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole2d_fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(kHole2DFusedMaxSmem)));
}

}  // namespace asdsm_b200
