// ASDSM iteration kernels for sm_100a (fp64).
//
// Every fine-grid pass reproduces the reference's arithmetic order so the residual and the
// merged skeleton are bitwise what proj/src computes for the same inputs:
//   A*u row dot    : proj/src/sparse.cpp:66-72 over the CSR order of fdm.cpp:110-117
//   residual       : proj/src/fdm.cpp:221-230
//   spline         : proj/src/spline.cpp:9-57
//   skeleton merge : proj/src/solver.cpp:154-196
//   hole rhs       : proj/src/solver.cpp:414-432
//   step control   : proj/src/solver.cpp:447-484, 621-677
// Reductions use a fixed grid and a fixed combine tree, so results are run-to-run
// deterministic (the reference's serial order is not reproduced).
#include <cmath>

#include "kernels.cuh"

#include <cstdlib>
#include "spline.cuh"
#include "ctrl.cuh"
#include "skel2d.cuh"

namespace asdsm_b200 {

long long g_kernel_launches = 0;

namespace {

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_down_sync(0xffffffffu, v, o));
  return v;
}

// Block-level reduction of up to 4 values (sum, max, sum, max); thread 0 writes partials.
__device__ void block_reduce4(double s0, double m1, double s2, double m3, double* partials) {
  __shared__ double sh[4][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  s0 = warp_sum(s0);
  m1 = warp_max(m1);
  s2 = warp_sum(s2);
  m3 = warp_max(m3);
  if (lane == 0) {
    sh[0][w] = s0;
    sh[1][w] = m1;
    sh[2][w] = s2;
    sh[3][w] = m3;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    s0 = lane < nw ? sh[0][lane] : 0.0;
    m1 = lane < nw ? sh[1][lane] : 0.0;
    s2 = lane < nw ? sh[2][lane] : 0.0;
    m3 = lane < nw ? sh[3][lane] : 0.0;
    s0 = warp_sum(s0);
    m1 = warp_max(m1);
    s2 = warp_sum(s2);
    m3 = warp_max(m3);
    if (lane == 0) {
      partials[0 * kRedStride + blockIdx.x] = s0;
      partials[1 * kRedStride + blockIdx.x] = m1;
      partials[2 * kRedStride + blockIdx.x] = s2;
      partials[3 * kRedStride + blockIdx.x] = m3;
    }
  }
}


struct StencilArgs {
  const double* u0;
  const double* u1;
  const double* e;
  const double* b;
  double* uo0;
  double* uo1;
  double* ro0;
  double* ro1;
  const double* exact;
  FineGeom g;
  Stencil st;
  double* partials;
  DevState* state;
  CtrlArgs ctrl;
  double* history;
};

// A*v at fine point (i,j,k) in the CSR column order of fdm.cpp:110-117, no contraction.
// V(q, axis, dir) returns v at neighbour q (axis -1 = the point itself).
template <int DIM, typename F>
__device__ __forceinline__ double apply_row(const FineGeom& g, const Stencil& st, i64 p, int i, int j, int k, F V,
                                            double& vp) {
  double acc = 0.0;
  if (DIM == 3 && k > 0) acc = add_rn(acc, mul_rn(st.left[2], V(p - g.stride[2], 2, -1)));
  if (j > 0) acc = add_rn(acc, mul_rn(st.left[1], V(p - g.stride[1], 1, -1)));
  if (i > 0) acc = add_rn(acc, mul_rn(st.left[0], V(p - 1, 0, -1)));
  vp = V(p, -1, 0);
  acc = add_rn(acc, mul_rn(st.diag, vp));
  if (i < g.ext[0] - 1 && st.has_right[0]) acc = add_rn(acc, mul_rn(st.right[0], V(p + 1, 0, 1)));
  if (j < g.ext[1] - 1 && st.has_right[1]) acc = add_rn(acc, mul_rn(st.right[1], V(p + g.stride[1], 1, 1)));
  if (DIM == 3 && k < g.ext[2] - 1 && st.has_right[2])
    acc = add_rn(acc, mul_rn(st.right[2], V(p + g.stride[2], 2, 1)));
  return acc;
}

// residual (UPDATE=false): r[cur] = b - A u[cur]
// update   (UPDATE=true) : u[1-cur] = u[cur] + s e ; r[1-cur] = b - A u[1-cur]
// plus per-block partials of sum r^2, max |r|, sum d^2, max |d| (d = u - exact).
template <int DIM, bool UPDATE>
__global__ void __launch_bounds__(kRedThreads) stencil_kernel(StencilArgs a) {
  DevState* S = a.state;
  if (!S->active) return;
  double s = 0.0;
  if (UPDATE) s = S->s;
  const bool work = !UPDATE || s != 0.0;
  const int cur = S->cur;
  const double* __restrict__ u = cur ? a.u1 : a.u0;
  double* __restrict__ uo = UPDATE ? (cur ? a.uo0 : a.uo1) : nullptr;
  double* __restrict__ ro = UPDATE ? (cur ? a.ro0 : a.ro1) : (cur ? a.ro1 : a.ro0);
  const double* __restrict__ e = a.e;
  const FineGeom& g = a.g;
  const int nseg = (g.ext[0] + blockDim.x - 1) / blockDim.x;
  const i64 rows = static_cast<i64>(g.ext[1]) * (DIM == 3 ? g.ext[2] : 1);
  const i64 items = rows * nseg;
  double ssq = 0.0, rmax = 0.0, esq = 0.0, emax = 0.0;
  auto V = [&](i64 q, int, int) -> double {
    if (UPDATE) return add_rn(u[q], mul_rn(s, e[q]));
    return u[q];
  };
  for (i64 it = work ? blockIdx.x : items; it < items; it += gridDim.x) {
    const i64 row = it / nseg;
    const int i = static_cast<int>((it % nseg) * blockDim.x + threadIdx.x);
    if (i >= g.ext[0]) continue;
    const int j = static_cast<int>(row % g.ext[1]);
    const int k = DIM == 3 ? static_cast<int>(row / g.ext[1]) : 0;
    const i64 p = i + row * g.stride[1];
    double vp;
    const double av = apply_row<DIM>(g, a.st, p, i, j, k, V, vp);
    const double r = sub_rn(a.b[p], av);
    ro[p] = r;
    if (UPDATE) uo[p] = vp;
    ssq += r * r;
    rmax = fmax(rmax, fabs(r));
    if (a.exact) {
      const double d = vp - a.exact[p];
      esq += d * d;
      emax = fmax(emax, fabs(d));
    }
  }
  block_reduce4(ssq, rmax, esq, emax, a.partials);
  fold_ctrl(a.ctrl, a.partials, S, a.history);
}

struct DotArgs {
  const double* e;
  const double* r0;
  const double* r1;
  FineGeom g;
  Stencil st;
  double* partials;
  DevState* state;
  CtrlArgs ctrl;
  double* history;
};

// w = A e (all rows, sparse.cpp:49-58 order); partial <r, w> and <w, w> (solver.cpp:456-461).
template <int DIM>
__global__ void __launch_bounds__(kRedThreads) ae_dots_kernel(DotArgs a) {
  DevState* S = a.state;
  if (!S->active) return;
  const bool work = S->have_e;
  const double* __restrict__ r = S->cur ? a.r1 : a.r0;
  const double* __restrict__ e = a.e;
  const FineGeom& g = a.g;
  const int nseg = (g.ext[0] + blockDim.x - 1) / blockDim.x;
  const i64 rows = static_cast<i64>(g.ext[1]) * (DIM == 3 ? g.ext[2] : 1);
  const i64 items = rows * nseg;
  double num = 0.0, den = 0.0;
  auto V = [&](i64 q, int, int) -> double { return e[q]; };
  for (i64 it = work ? blockIdx.x : items; it < items; it += gridDim.x) {
    const i64 row = it / nseg;
    const int i = static_cast<int>((it % nseg) * blockDim.x + threadIdx.x);
    if (i >= g.ext[0]) continue;
    const int j = static_cast<int>(row % g.ext[1]);
    const int k = DIM == 3 ? static_cast<int>(row / g.ext[1]) : 0;
    const i64 p = i + row * g.stride[1];
    double vp;
    const double w = apply_row<DIM>(g, a.st, p, i, j, k, V, vp);
    num += r[p] * w;
    den += w * w;
  }
  block_reduce4(num, 0.0, den, 0.0, a.partials);
  fold_ctrl(a.ctrl, a.partials, S, a.history);
}

// Restriction r -> one tensor submesh (Projector::apply with build_projector's map,
// mesh.cpp:174-179, 226-255).
__global__ void gather_kernel(const double* src0, const double* src1, double* dst, MeshDev m, unsigned mask, i64 count,
                              const DevState* state) {
  if (!state->active) return;
  const double* src = state->cur ? src1 : src0;
  int ext[3];
  i64 fstride[3];
  i64 s = 1;
  for (int a = 0; a < 3; ++a) {
    ext[a] = a < m.dim ? (((mask >> a) & 1u) ? m.nc[a] : m.nf[a]) : 1;
    fstride[a] = s;
    s *= a < m.dim ? m.nf[a] : 1;
  }
  if (count < (i64{1} << 31)) {  // 32-bit index arithmetic (three 64-bit divisions per point otherwise)
    const unsigned n = static_cast<unsigned>(count), e0 = ext[0], e1 = ext[1];
    for (unsigned t = blockIdx.x * blockDim.x + threadIdx.x; t < n; t += gridDim.x * blockDim.x) {
      const unsigned q0 = t / e0, i0 = t - q0 * e0, q1 = q0 / e1, i1 = q0 - q1 * e1, i2 = q1;
      const unsigned ia[3] = {i0, i1, i2};
      i64 f = 0;
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const i64 fi = ((mask >> a) & 1u) ? static_cast<i64>(ia[a] + 1) * m.n[a] - 1 : ia[a];
        if (a < m.dim) f += fi * fstride[a];
      }
      dst[t] = src[f];
    }
    return;
  }
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < count;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    i64 rem = t, f = 0;
    for (int a = 0; a < m.dim; ++a) {
      const int ia = static_cast<int>(rem % ext[a]);
      rem /= ext[a];
      const i64 fi = ((mask >> a) & 1u) ? static_cast<i64>(ia + 1) * m.n[a] - 1 : ia;
      f += fi * fstride[a];
    }
    dst[t] = src[f];
  }
}

__global__ void __launch_bounds__(kRedThreads) norm_sq_kernel(const double* x, i64 n, double* partials,
                                                             DevState* state, CtrlArgs c, double* history) {
  if (!state->active) return;
  double s = 0.0;
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<i64>(gridDim.x) * blockDim.x)
    s += x[t] * x[t];
  block_reduce4(s, 0.0, 0.0, 0.0, partials);
  fold_ctrl(c, partials, state, history);
}

// normalize_or_throw (solver.cpp:79-84): v /= ||v||_2 element by element.
__global__ void divide_kernel(double* x, i64 n, const double* divisor, const DevState* state) {
  if (!state->active || !state->have_e) return;
  const double d = *divisor;
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < n;
       t += static_cast<i64>(gridDim.x) * blockDim.x)
    x[t] = x[t] / d;
}

// ---------------------------------------------------------------- 2D skeleton --------------
// Phase 1: cross values u_hat (Richardson u1 + u2 - u_cc, or the seeded choice) and the
// corrections e1 = u_hat - P u_fc, e2 = u_hat - P u_cf (solver.cpp:166-184).
__global__ void skel2d_cc_kernel(Skel2DArgs a, const DevState* state) {
  if (!state->active || !state->have_e) return;
  const MeshDev& m = a.m;
  const int ncc = m.nc[0] * m.nc[1];
  for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < ncc; t += gridDim.x * blockDim.x) {
    const int I = t % m.nc[0], J = t / m.nc[0];
    double u1 = a.u_fc[static_cast<i64>((I + 1) * m.n[0] - 1) + static_cast<i64>(m.nf[0]) * J];
    double u2 = a.u_cf[I + static_cast<i64>(m.nc[0]) * ((J + 1) * m.n[1] - 1)];
    if (a.norm_fc) {
      u1 = u1 / *a.norm_fc;
      u2 = u2 / *a.norm_cf;
    }
    double uh;
    if (a.u_cc) {
      uh = __dsub_rn(__dadd_rn(u1, u2), a.u_cc[t]);
    } else {
      uh = (a.coin[0] == 0) ? u2 : u1;
    }
    a.e1[t] = __dsub_rn(uh, u1);
    a.e2[t] = __dsub_rn(uh, u2);
  }
}

// Phase 2: spline second derivatives, one thread per coarse line.
__global__ void skel2d_spline_kernel(Skel2DArgs a, double* work, const DevState* state) {
  if (!state->active || !state->have_e) return;
  const MeshDev& m = a.m;
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  const int nlines = m.nc[1] + m.nc[0];
  if (t >= nlines) return;
  const int maxn = (m.nc[0] > m.nc[1] ? m.nc[0] : m.nc[1]) + 2;
  double* y = work + static_cast<i64>(t) * 4 * maxn;
  double* dg = y + maxn;
  double* up = dg + maxn;
  double* rh = up + maxn;
  if (t < m.nc[1]) {  // line J along x through e1[:, J]
    const int J = t;
    const int nc = m.nc[0];
    y[0] = 0.0;
    for (int C = 0; C < nc; ++C) y[C + 1] = a.e1[C + static_cast<i64>(nc) * J];
    y[nc + 1] = 0.0;
    spline_second_derivs(m, 0, y, a.m1 + static_cast<i64>(J) * (nc + 2), dg, up, rh);
  } else {  // line I along y through e2[I, :]
    const int I = t - m.nc[1];
    const int nc = m.nc[1];
    y[0] = 0.0;
    for (int C = 0; C < nc; ++C) y[C + 1] = a.e2[I + static_cast<i64>(m.nc[0]) * C];
    y[nc + 1] = 0.0;
    spline_second_derivs(m, 1, y, a.m2 + static_cast<i64>(I) * (nc + 2), dg, up, rh);
  }
}

// Phases 1+2 in one CTA (coarse counts <= 62): cross values, corrections, spline second
// derivatives with per-thread local arrays.
__global__ void skel2d_ccspline_kernel(Skel2DArgs a, const DevState* state) {
  if (!state->active || !state->have_e) return;
  const MeshDev& m = a.m;
  const int nc0 = m.nc[0], nc1 = m.nc[1];
  for (int t = threadIdx.x; t < nc0 * nc1; t += blockDim.x) {
    const int I = t % nc0, J = t / nc0;
    double u1 = a.u_fc[static_cast<i64>((I + 1) * m.n[0] - 1) + static_cast<i64>(m.nf[0]) * J];
    double u2 = a.u_cf[I + static_cast<i64>(nc0) * ((J + 1) * m.n[1] - 1)];
    if (a.norm_fc) {
      u1 = u1 / *a.norm_fc;
      u2 = u2 / *a.norm_cf;
    }
    double uh;
    if (a.u_cc) uh = __dsub_rn(__dadd_rn(u1, u2), a.u_cc[t]);
    else uh = (a.coin[0] == 0) ? u2 : u1;
    a.e1[t] = __dsub_rn(uh, u1);
    a.e2[t] = __dsub_rn(uh, u2);
  }
  __syncthreads();
  constexpr int KM = 64;
  for (int t = threadIdx.x; t < nc0 + nc1; t += blockDim.x) {
    double y[KM], dg[KM], up[KM], rh[KM];
    if (t < nc1) {
      const int J = t;
      y[0] = 0.0;
      for (int C = 0; C < nc0; ++C) y[C + 1] = a.e1[C + static_cast<i64>(nc0) * J];
      y[nc0 + 1] = 0.0;
      spline_second_derivs(m, 0, y, a.m1 + static_cast<i64>(J) * (nc0 + 2), dg, up, rh);
    } else {
      const int I = t - nc1;
      y[0] = 0.0;
      for (int C = 0; C < nc1; ++C) y[C + 1] = a.e2[I + static_cast<i64>(nc0) * C];
      y[nc1 + 1] = 0.0;
      spline_second_derivs(m, 1, y, a.m2 + static_cast<i64>(I) * (nc1 + 2), dg, up, rh);
    }
  }
}

// Phase 3: corrected anisotropic values merged onto the skeleton points (solver.cpp:186-195):
//   coarse-row points  : ut_fc = u_fc + S1_J(x_i)
//   coarse-column points: ut_cf = u_cf + S2_I(y_j)
//   cross points       : (0 + ut_fc) + ut_cf + (-ut_cf), the scatter_add sequence.
__global__ void skel2d_write_kernel(Skel2DArgs a, const DevState* state) {
  if (!state->active || !state->have_e) return;
  const MeshDev& m = a.m;
  const int nc0 = m.nc[0], nc1 = m.nc[1];
  const i64 nrow_pts = static_cast<i64>(nc1) * m.nf[0];
  const i64 ncol_pts = static_cast<i64>(nc0) * m.nf[1];
  auto ut_cf = [&](int I, int j) {
    const double* mm2 = a.m2 + static_cast<i64>(I) * (nc1 + 2);
    auto y2 = [&](int c) -> double { return (c == 0 || c == nc1 + 1) ? 0.0 : a.e2[I + static_cast<i64>(nc0) * (c - 1)]; };
    double u = a.u_cf[I + static_cast<i64>(nc0) * j];
    if (a.norm_cf) u = u / *a.norm_cf;
    return __dadd_rn(u, spline_eval(m, 1, y2, mm2, j + 1));
  };
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < nrow_pts + ncol_pts;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    if (t < nrow_pts) {
      const int i = static_cast<int>(t % m.nf[0]);
      const int J = static_cast<int>(t / m.nf[0]);
      const int j = (J + 1) * m.n[1] - 1;
      const double* mm1 = a.m1 + static_cast<i64>(J) * (nc0 + 2);
      auto y1 = [&](int c) -> double { return (c == 0 || c == nc0 + 1) ? 0.0 : a.e1[(c - 1) + static_cast<i64>(nc0) * J]; };
      double ufc = a.u_fc[i + static_cast<i64>(m.nf[0]) * J];
      if (a.norm_fc) ufc = ufc / *a.norm_fc;
      const double av = __dadd_rn(ufc, spline_eval(m, 0, y1, mm1, i + 1));
      double val = av;
      if ((i + 1) % m.n[0] == 0) {
        const double bv = ut_cf((i + 1) / m.n[0] - 1, j);
        val = __dadd_rn(__dadd_rn(av, bv), -bv);
      }
      a.out[i + static_cast<i64>(m.nf[0]) * j] = val;
    } else {
      const i64 tc = t - nrow_pts;
      const int j = static_cast<int>(tc % m.nf[1]);
      const int I = static_cast<int>(tc / m.nf[1]);
      if ((j + 1) % m.n[1] == 0) continue;  // cross points are written by the row pass
      const int i = (I + 1) * m.n[0] - 1;
      a.out[i + static_cast<i64>(m.nf[0]) * j] = ut_cf(I, j);
    }
  }
}

// Hole right-hand side (solver.cpp:416-424): rhs_p = b_p - (A_ff * skeleton)_p for every
// hole point p, written in place of the (zero) skeleton value.  Hole neighbours carry 0.
template <int DIM>
__global__ void hole_rhs_kernel(double* e, const double* b, FineGeom g, Stencil st, MeshDev m, const DevState* state) {
  if (!state->active || !state->have_e) return;
  const int nseg = (g.ext[0] + blockDim.x - 1) / blockDim.x;
  const i64 rows = static_cast<i64>(g.ext[1]) * (DIM == 3 ? g.ext[2] : 1);
  const i64 items = rows * nseg;
  for (i64 it = blockIdx.x; it < items; it += gridDim.x) {
    const i64 row = it / nseg;
    const int i = static_cast<int>((it % nseg) * blockDim.x + threadIdx.x);
    if (i >= g.ext[0]) continue;
    const int j = static_cast<int>(row % g.ext[1]);
    const int k = DIM == 3 ? static_cast<int>(row / g.ext[1]) : 0;
    const bool sk_i = (i + 1) % m.n[0] == 0, sk_j = (j + 1) % m.n[1] == 0;
    const bool sk_k = DIM == 3 ? ((k + 1) % m.n[2] == 0) : false;
    if (sk_i || sk_j || sk_k) continue;  // skeleton point
    const i64 p = i + row * g.stride[1];
    // Neighbour q is a skeleton point iff its moved coordinate lies on a coarse plane
    // (the unmoved coordinates are hole coordinates); hole neighbours carry 0.
    const int idx[3] = {i, j, k};
    auto V = [&](i64 q, int axis, int dir) -> double {
      if (axis < 0) return 0.0;
      return ((idx[axis] + dir + 1) % m.n[axis] == 0) ? e[q] : 0.0;
    };
    double vp;
    const double av = apply_row<DIM>(g, st, p, i, j, k, V, vp);
    const double bp = b ? b[p] : 0.0;
    e[p] = sub_rn(bp, av);
  }
}

// Same result, one CTA per fine row (j, k): the row's skeleton tests are row-uniform and the
// x test is one 32-bit remainder per point (the generic kernel above spends ~10 64-bit
// divisions per point).  Identical arithmetic (apply_row, hole neighbours carry 0).
template <int DIM>
__global__ void __launch_bounds__(256) hole_rhs_rows_kernel(double* e, const double* b, FineGeom g, Stencil st, MeshDev m,
                                                            const DevState* state) {
  if (!state->active || !state->have_e) return;
  const i64 rows = static_cast<i64>(g.ext[1]) * (DIM == 3 ? g.ext[2] : 1);
  for (i64 row = blockIdx.x; row < rows; row += gridDim.x) {
    const int j = static_cast<int>(row % g.ext[1]);
    const int k = DIM == 3 ? static_cast<int>(row / g.ext[1]) : 0;
    const int rj = j % m.n[1], rk = DIM == 3 ? k % m.n[2] : 0;
    if (rj == m.n[1] - 1 || (DIM == 3 && rk == m.n[2] - 1)) continue;  // skeleton row
    for (int i = threadIdx.x; i < g.ext[0]; i += blockDim.x) {
      const int ri = i % m.n[0];
      if (ri == m.n[0] - 1) continue;  // skeleton point
      const i64 p = i + row * g.stride[1];
      // neighbour along `axis` in direction dir is a skeleton point iff (idx + dir + 1) % n == 0
      auto V = [&](i64 q, int axis, int dir) -> double {
        if (axis < 0) return 0.0;
        const int r = axis == 0 ? ri : (axis == 1 ? rj : rk);
        const int n = m.n[axis];
        const bool sk = dir < 0 ? r == 0 : r == n - 2;
        return sk ? e[q] : 0.0;
      };
      double vp;
      const double av = apply_row<DIM>(g, st, p, i, j, k, V, vp);
      const double bp = b ? b[p] : 0.0;
      e[p] = sub_rn(bp, av);
    }
  }
}

__global__ void dense_matvec_kernel(const double* A, const double* b, double* x, int n, const DevState* state) {
  if (!state->active) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = blockDim.x >> 5;
  for (int i = blockIdx.x * nw + warp; i < n; i += gridDim.x * nw) {
    double s = 0.0;
    for (int j = lane; j < n; j += 32) s = fma(A[static_cast<i64>(i) * n + j], b[j], s);
    s = warp_sum(s);
    if (lane == 0) x[i] = s;
  }
}

}  // namespace

__global__ void state_init_kernel(DevState* S, int active, int have_e) {
  DevState h{};
  h.cur = 0;
  h.active = active;
  h.have_e = have_e;
  unsigned long long tns;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tns));
  h.t0_ns = static_cast<double>(tns);
  *S = h;
}

// Busy-waits on the global timer: queued ahead of a timed loop so the host enqueues every
// launch while the device is still busy (the loop is then timed device-side, not host-bound).
__global__ void spin_kernel(unsigned long long ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  do {
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  } while (t - t0 < ns);
}

__global__ void publish_copy_kernel(const DevState* S, double* u0, const double* u1, double* r0,
                                    const double* r1, i64 n) {
  if (S->cur == 0) return;
  const i64 stride = static_cast<i64>(gridDim.x) * blockDim.x;
  const i64 n2 = n / 2;
  for (i64 i = blockIdx.x * static_cast<i64>(blockDim.x) + threadIdx.x; i < n2; i += stride) {
    reinterpret_cast<double2*>(u0)[i] = reinterpret_cast<const double2*>(u1)[i];
    reinterpret_cast<double2*>(r0)[i] = reinterpret_cast<const double2*>(r1)[i];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) {
    u0[n - 1] = u1[n - 1];
    r0[n - 1] = r1[n - 1];
  }
}

__global__ void publish_flip_kernel(DevState* S) { S->cur = 0; }

void launch_publish(DevState* state, double* u0, const double* u1, double* r0, const double* r1, i64 n,
                    cudaStream_t s) {
  publish_copy_kernel<<<4 * 148, 256, 0, s>>>(state, u0, u1, r0, r1, n);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  publish_flip_kernel<<<1, 1, 0, s>>>(state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  g_kernel_launches += 2;
}

// measured (config 1): PDL overlaps kernel boundaries well on plain stream launches (1.46 ->
// 1.37 ms) but costs inside the captured graph (1.28 -> 1.32 ms), which is the faster of the
// two -- so it is opt-in (ASDSM_PDL=1)
bool pdl_enabled() {
  const bool on = std::getenv("ASDSM_PDL") != nullptr;
  return on;
}

void launch_spin(double us, cudaStream_t s) {
  spin_kernel<<<1, 1, 0, s>>>(static_cast<unsigned long long>(us * 1000.0));
  ASDSM_CUDA_CHECK(cudaGetLastError());
}

void launch_state_init(DevState* state, int active, int have_e, cudaStream_t s) {
  state_init_kernel<<<1, 1, 0, s>>>(state, active, have_e);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_stencil(int dim, bool update, const double* u0, const double* u1, const double* e, const double* b,
                    double* uo0, double* uo1, double* ro0, double* ro1, const double* exact, const FineGeom& g,
                    const Stencil& st, double* partials, DevState* state, cudaStream_t s, const CtrlArgs* ctrl,
                    double* history) {
  CtrlArgs c{};
  c.op = -1;
  if (ctrl) c = *ctrl;
  StencilArgs a{u0, u1, e, b, uo0, uo1, ro0, ro1, exact, g, st, partials, state, c, history};
  if (dim == 2) {
    if (update) stencil_kernel<2, true><<<kRedBlocks, kRedThreads, 0, s>>>(a);
    else stencil_kernel<2, false><<<kRedBlocks, kRedThreads, 0, s>>>(a);
  } else {
    if (update) stencil_kernel<3, true><<<kRedBlocks, kRedThreads, 0, s>>>(a);
    else stencil_kernel<3, false><<<kRedBlocks, kRedThreads, 0, s>>>(a);
  }
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_ae_dots(int dim, const double* e, const double* r0, const double* r1, const FineGeom& g,
                    const Stencil& st, double* partials, DevState* state, cudaStream_t s, const CtrlArgs* ctrl,
                    double* history) {
  CtrlArgs c{};
  c.op = -1;
  if (ctrl) c = *ctrl;
  DotArgs a{e, r0, r1, g, st, partials, state, c, history};
  if (dim == 2) ae_dots_kernel<2><<<kRedBlocks, kRedThreads, 0, s>>>(a);
  else ae_dots_kernel<3><<<kRedBlocks, kRedThreads, 0, s>>>(a);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_gather(const double* src0, const double* src1, double* dst, const MeshDev& m, unsigned mask, i64 count,
                   DevState* state, cudaStream_t s) {
  const int bs = 256;
  const int per_sm = std::getenv("ASDSM_GATHER_CTAS") ? std::atoi(std::getenv("ASDSM_GATHER_CTAS")) : 4;  // 8 and 12 measured the same
  const i64 nb = std::min<i64>((count + bs - 1) / bs, static_cast<i64>(per_sm) * kNumSms);
  gather_kernel<<<static_cast<unsigned>(nb), bs, 0, s>>>(src0, src1, dst, m, mask, count, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_norm_sq(const double* x, i64 n, double* partials, DevState* state, cudaStream_t s, const CtrlArgs* ctrl,
                    double* history) {
  CtrlArgs c{};
  c.op = -1;
  if (ctrl) c = *ctrl;
  norm_sq_kernel<<<kRedBlocks, kRedThreads, 0, s>>>(x, n, partials, state, c, history);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_divide(double* x, i64 n, const double* divisor, DevState* state, cudaStream_t s) {
  const int bs = 256;
  const i64 nb = std::min<i64>((n + bs - 1) / bs, 4 * kNumSms);
  divide_kernel<<<static_cast<unsigned>(nb), bs, 0, s>>>(x, n, divisor, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_ctrl(const CtrlArgs& a, const double* partials, DevState* state, double* history, cudaStream_t s) {
  ctrl_kernel<<<1, kRedThreads, 0, s>>>(a, partials, state, history);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_skeleton2d(const Skel2DArgs& a, DevState* state, cudaStream_t s) {
  if (a.m.nc[0] <= 62 && a.m.nc[1] <= 62) {
    skel2d_ccspline_kernel<<<1, 256, 0, s>>>(a, state);
    ASDSM_CUDA_CHECK(cudaGetLastError());
    const i64 npts = static_cast<i64>(a.m.nc[1]) * a.m.nf[0] + static_cast<i64>(a.m.nc[0]) * a.m.nf[1];
    const i64 nb = std::min<i64>((npts + 255) / 256, 4 * kNumSms);
    skel2d_write_kernel<<<static_cast<unsigned>(nb), 256, 0, s>>>(a, state);
    ASDSM_CUDA_CHECK(cudaGetLastError());
    g_kernel_launches += 2;
    return;
  }
  const int ncc = a.m.nc[0] * a.m.nc[1];
  g_kernel_launches += 2;
  skel2d_cc_kernel<<<(ncc + 255) / 256, 256, 0, s>>>(a, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  const int nlines = a.m.nc[0] + a.m.nc[1];
  // spline work: 4 * (max nc + 2) doubles per line; lives after m2 in the same allocation
  const int maxn = (a.m.nc[0] > a.m.nc[1] ? a.m.nc[0] : a.m.nc[1]) + 2;
  double* work = a.m2 + static_cast<i64>(a.m.nc[0]) * (a.m.nc[1] + 2);
  (void)maxn;
  skel2d_spline_kernel<<<(nlines + 63) / 64, 64, 0, s>>>(a, work, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  const i64 npts = static_cast<i64>(a.m.nc[1]) * a.m.nf[0] + static_cast<i64>(a.m.nc[0]) * a.m.nf[1];
  const i64 nb = std::min<i64>((npts + 255) / 256, 4 * kNumSms);
  skel2d_write_kernel<<<static_cast<unsigned>(nb), 256, 0, s>>>(a, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

namespace {

__global__ void skel2d_ccspline_fast_kernel(Skel2DArgs a, const DevState* state) {
  if (!state->active || !state->have_e) return;
  skel2d_ccspline_block(a);
}

// skeleton points from the precomputed segment coefficients (no divisions per point)
__global__ void skel2d_write_fast_kernel(Skel2DArgs a, const DevState* state) {
  if (!state->active || !state->have_e) return;
  const MeshDev& m = a.m;
  const int nc0 = m.nc[0], nc1 = m.nc[1];
  const double nfc = a.norm_fc ? *a.norm_fc : 1.0;
  const double ncf = a.norm_cf ? *a.norm_cf : 1.0;
  const i64 nrow_pts = static_cast<i64>(nc1) * m.nf[0];
  const i64 ncol_pts = static_cast<i64>(nc0) * m.nf[1];
  auto ut_cf = [&](int I, int j) {
    double u = a.u_cf[I + static_cast<i64>(nc0) * j];
    if (a.norm_cf) u = u / ncf;
    return __dadd_rn(u, skel_seg_eval(a.sp_tab[1], a.seg2 + static_cast<i64>(I) * 4 * (nc1 + 1), nc1, m.n[1], m.h[1], j + 1));
  };
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < nrow_pts + ncol_pts;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    if (t < nrow_pts) {
      const int i = static_cast<int>(t % m.nf[0]);
      const int J = static_cast<int>(t / m.nf[0]);
      const int j = (J + 1) * m.n[1] - 1;
      double ufc = a.u_fc[i + static_cast<i64>(m.nf[0]) * J];
      if (a.norm_fc) ufc = ufc / nfc;
      const double av = __dadd_rn(ufc, skel_seg_eval(a.sp_tab[0], a.seg1 + static_cast<i64>(J) * 4 * (nc0 + 1), nc0,
                                                     m.n[0], m.h[0], i + 1));
      double val = av;
      if ((i + 1) % m.n[0] == 0) {
        const double bv = ut_cf((i + 1) / m.n[0] - 1, j);
        val = __dadd_rn(__dadd_rn(av, bv), -bv);
      }
      a.out[i + static_cast<i64>(m.nf[0]) * j] = val;
    } else {
      const i64 tc = t - nrow_pts;
      const int j = static_cast<int>(tc % m.nf[1]);
      const int I = static_cast<int>(tc / m.nf[1]);
      if ((j + 1) % m.n[1] == 0) continue;
      const int i = (I + 1) * m.n[0] - 1;
      a.out[i + static_cast<i64>(m.nf[0]) * j] = ut_cf(I, j);
    }
  }
}

}  // namespace

void launch_skel2d_ccspline_fast(const Skel2DArgs& a, DevState* state, cudaStream_t s) {
  skel2d_ccspline_fast_kernel<<<1, 256, 0, s>>>(a, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_skel2d_write_fast(const Skel2DArgs& a, DevState* state, cudaStream_t s) {
  const i64 npts = static_cast<i64>(a.m.nc[1]) * a.m.nf[0] + static_cast<i64>(a.m.nc[0]) * a.m.nf[1];
  const i64 nb = std::min<i64>((npts + 255) / 256, 4 * kNumSms);
  skel2d_write_fast_kernel<<<static_cast<unsigned>(nb), 256, 0, s>>>(a, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

// zero_clamped_spline + CubicSpline ctor (spline.cpp:9-37, 58-76): the knot-only terms, in
// the reference's operation order (host compiled with -ffp-contract=off).
// The skeleton correction along one axis is linear in the cross-point corrections: value at
// fine index i = sum_I B[i][I] y_I for the zero-clamped natural spline through (0, 0), the
// stations (y_I) and (1, 0) (spline.cpp).  B, evaluated exactly like spline_axis_table +
// skel_seg_eval but in long double, turns the per-iteration spline phase into a small GEMM.
std::vector<double> spline_basis_table(int nc, int n, double h, int nf) {
  using ld = long double;
  const int np = nc + 2, ni = nc;
  std::vector<ld> x(static_cast<size_t>(np));
  x[0] = 0.0L;
  for (int c = 1; c <= nc; ++c) x[static_cast<size_t>(c)] = static_cast<ld>(static_cast<double>(static_cast<long long>(c) * n) * h);
  x[static_cast<size_t>(np - 1)] = 1.0L;
  std::vector<double> B(static_cast<size_t>(nf) * nc, 0.0);
  for (int I = 0; I < nc; ++I) {
    std::vector<ld> y(static_cast<size_t>(np), 0.0L), m(static_cast<size_t>(np), 0.0L);
    y[static_cast<size_t>(I + 1)] = 1.0L;
    // (hl/6) m_i + ((hl + hr)/3) m_{i+1} + (hr/6) m_{i+2} = rhs_i, m_0 = m_{np-1} = 0
    std::vector<ld> a(static_cast<size_t>(ni)), d(static_cast<size_t>(ni)), c(static_cast<size_t>(ni)), r(static_cast<size_t>(ni));
    for (int i = 0; i < ni; ++i) {
      const ld hl = x[static_cast<size_t>(i + 1)] - x[static_cast<size_t>(i)];
      const ld hr = x[static_cast<size_t>(i + 2)] - x[static_cast<size_t>(i + 1)];
      a[static_cast<size_t>(i)] = hl / 6.0L;
      d[static_cast<size_t>(i)] = (hl + hr) / 3.0L;
      c[static_cast<size_t>(i)] = hr / 6.0L;
      r[static_cast<size_t>(i)] = (y[static_cast<size_t>(i + 2)] - y[static_cast<size_t>(i + 1)]) / hr -
                                  (y[static_cast<size_t>(i + 1)] - y[static_cast<size_t>(i)]) / hl;
    }
    for (int i = 1; i < ni; ++i) {
      const ld wi = a[static_cast<size_t>(i)] / d[static_cast<size_t>(i - 1)];
      d[static_cast<size_t>(i)] -= wi * c[static_cast<size_t>(i - 1)];
      r[static_cast<size_t>(i)] -= wi * r[static_cast<size_t>(i - 1)];
    }
    for (int i = ni - 1; i >= 0; --i)
      m[static_cast<size_t>(i + 1)] = (r[static_cast<size_t>(i)] - (i + 1 < ni ? c[static_cast<size_t>(i)] * m[static_cast<size_t>(i + 2)] : 0.0L)) /
                                      d[static_cast<size_t>(i)];
    for (int i = 0; i < nf; ++i) {
      const int fi = i + 1;
      int cs = fi / n;
      if (cs > nc) cs = nc;
      const ld hs = x[static_cast<size_t>(cs + 1)] - x[static_cast<size_t>(cs)];
      const ld c1 = (y[static_cast<size_t>(cs + 1)] - y[static_cast<size_t>(cs)]) / hs -
                    hs * (2.0L * m[static_cast<size_t>(cs)] + m[static_cast<size_t>(cs + 1)]) / 6.0L;
      const ld c2 = m[static_cast<size_t>(cs)] / 2.0L;
      const ld c3 = (m[static_cast<size_t>(cs + 1)] - m[static_cast<size_t>(cs)]) / (6.0L * hs);
      const ld t = static_cast<ld>(static_cast<double>(fi) * h) - x[static_cast<size_t>(cs)];
      const ld v = y[static_cast<size_t>(cs)] + t * (c1 + t * (c2 + t * c3));
      B[static_cast<size_t>(i) * nc + I] = static_cast<double>(v);
    }
  }
  return B;
}

std::vector<double> spline_axis_table(int nc, int n, double h) {
  const int np = nc + 2, ni = nc;
  std::vector<double> x(static_cast<size_t>(np));
  x[0] = 0.0;
  for (int c = 1; c <= nc; ++c) x[static_cast<size_t>(c)] = static_cast<double>(static_cast<long long>(c) * n) * h;
  x[static_cast<size_t>(np - 1)] = 1.0;
  std::vector<double> hl(static_cast<size_t>(ni)), hr(static_cast<size_t>(ni)), w(static_cast<size_t>(ni), 0.0),
      dg(static_cast<size_t>(ni)), up(static_cast<size_t>(ni));
  for (int i = 0; i < ni; ++i) {
    hl[static_cast<size_t>(i)] = x[static_cast<size_t>(i + 1)] - x[static_cast<size_t>(i)];
    hr[static_cast<size_t>(i)] = x[static_cast<size_t>(i + 2)] - x[static_cast<size_t>(i + 1)];
    dg[static_cast<size_t>(i)] = (hl[static_cast<size_t>(i)] + hr[static_cast<size_t>(i)]) / 3.0;
    up[static_cast<size_t>(i)] = hr[static_cast<size_t>(i)] / 6.0;
  }
  for (int i = 1; i < ni; ++i) {
    const double lower = (x[static_cast<size_t>(i + 1)] - x[static_cast<size_t>(i)]) / 6.0;
    const double wi = lower / dg[static_cast<size_t>(i - 1)];
    w[static_cast<size_t>(i)] = wi;
    dg[static_cast<size_t>(i)] -= wi * up[static_cast<size_t>(i - 1)];
  }
  std::vector<double> tab;
  tab.insert(tab.end(), x.begin(), x.end());
  tab.insert(tab.end(), hl.begin(), hl.end());
  tab.insert(tab.end(), hr.begin(), hr.end());
  tab.insert(tab.end(), w.begin(), w.end());
  tab.insert(tab.end(), dg.begin(), dg.end());
  tab.insert(tab.end(), up.begin(), up.end());
  return tab;
}

namespace {

template <int DIM>
__global__ void __launch_bounds__(kRedThreads) subsample_dots_kernel(const long long* rows, int nrows, const double* e,
                                                                      const double* r0, const double* r1, FineGeom g,
                                                                      Stencil st, double* partials, DevState* S,
                                                                      double* history, CtrlArgs c, const double* coef) {
  if (!S->active) return;
  const double* r = S->cur ? r1 : r0;
  double num = 0.0, den = 0.0;
  if (S->have_e) {
    auto V = [&](i64 q, int, int) -> double { return e[q]; };
    for (int t = blockIdx.x * blockDim.x + threadIdx.x; t < nrows; t += gridDim.x * blockDim.x) {
      const i64 p = rows[t];
      const int i = static_cast<int>(p % g.ext[0]);
      const int j = static_cast<int>((p / g.ext[0]) % g.ext[1]);
      const int k = DIM == 3 ? static_cast<int>(p / (static_cast<i64>(g.ext[0]) * g.ext[1])) : 0;
      double w;
      if (coef) {  // per-point coefficients, same CSR order
        const int idx[3] = {i, j, k};
        double acc = 0.0;
        int slot = 0;
        for (int a = DIM - 1; a >= 0; --a, ++slot)
          if (idx[a] > 0) acc = __dadd_rn(acc, __dmul_rn(coef[slot * g.size + p], e[p - g.stride[a]]));
        acc = __dadd_rn(acc, __dmul_rn(coef[slot * g.size + p], e[p]));
        ++slot;
        for (int a = 0; a < DIM; ++a, ++slot)
          if (idx[a] < g.ext[a] - 1 && st.has_right[a]) acc = __dadd_rn(acc, __dmul_rn(coef[slot * g.size + p], e[p + g.stride[a]]));
        w = acc;
      } else {
        double vp;
        w = apply_row<DIM>(g, st, p, i, j, k, V, vp);
      }
      num += r[p] * w;
      den += w * w;
    }
  }
  block_reduce4_march(num, 0.0, den, 0.0, partials);
  fold_ctrl(c, partials, S, history);
}

}  // namespace

void launch_subsample_dots(int dim, const long long* rows, int nrows, const double* e, const double* r0,
                           const double* r1, const FineGeom& g, const Stencil& st, double* partials,
                           DevState* state, double* history, cudaStream_t s, const double* coef) {
  CtrlArgs c{};
  c.op = kCtrlSubDots;
  const unsigned nb = static_cast<unsigned>(std::max(1, std::min((nrows + 255) / 256, kRedBlocks)));
  if (dim == 2)
    subsample_dots_kernel<2><<<nb, kRedThreads, 0, s>>>(rows, nrows, e, r0, r1, g, st, partials, state, history, c, coef);
  else
    subsample_dots_kernel<3><<<nb, kRedThreads, 0, s>>>(rows, nrows, e, r0, r1, g, st, partials, state, history, c, coef);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_hole_rhs(int dim, double* e, const double* b, const FineGeom& g, const Stencil& st, const MeshDev& m,
                     DevState* state, cudaStream_t s) {
  if (std::getenv("ASDSM_HOLE_RHS_OLD") != nullptr) {  // (read at capture time)
    if (dim == 2) hole_rhs_kernel<2><<<kRedBlocks, kRedThreads, 0, s>>>(e, b, g, st, m, state);
    else hole_rhs_kernel<3><<<kRedBlocks, kRedThreads, 0, s>>>(e, b, g, st, m, state);
  } else {
    const i64 rows = static_cast<i64>(g.ext[1]) * (dim == 3 ? g.ext[2] : 1);
    const unsigned nb = static_cast<unsigned>(std::min<i64>(rows, 32LL * kNumSms));
    const int bs = g.ext[0] >= 256 ? 256 : 128;
    if (dim == 2) hole_rhs_rows_kernel<2><<<nb, bs, 0, s>>>(e, b, g, st, m, state);
    else hole_rhs_rows_kernel<3><<<nb, bs, 0, s>>>(e, b, g, st, m, state);
  }
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_dense_matvec(const double* Ainv, const double* b, double* x, int n, DevState* state, cudaStream_t s) {
  dense_matvec_kernel<<<(n + 7) / 8, 256, 0, s>>>(Ainv, b, x, n, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200

namespace asdsm_b200 {
namespace {

__global__ void projector_map_kernel(MeshDev m, unsigned from_mask, unsigned to_mask, long long* out, i64 count) {
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < count;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    i64 rem = t, src = 0, fstride = 1;
    for (int a = 0; a < m.dim; ++a) {
      const bool tc = (to_mask >> a) & 1u, fc = (from_mask >> a) & 1u;
      const int text = tc ? m.nc[a] : m.nf[a];
      const int fext = fc ? m.nc[a] : m.nf[a];
      const i64 ta = rem % text + 1;
      rem /= text;
      const i64 step = (tc && !fc) ? m.n[a] : 1;
      src += (ta * step - 1) * fstride;
      fstride *= fext;
    }
    out[t] = src;
  }
}

__global__ void hole_map_kernel(MeshDev m, long long* out, i64 count) {
  i64 per = 1;
  for (int a = 0; a < m.dim; ++a) per *= m.n[a] - 1;
  for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < count;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    i64 blk = t / per, in = t % per, lin = 0, fstride = 1;
    for (int a = 0; a < m.dim; ++a) {
      const i64 h = blk % (m.nc[a] + 1);
      blk /= (m.nc[a] + 1);
      const i64 k = in % (m.n[a] - 1) + 1;
      in /= (m.n[a] - 1);
      lin += (h * m.n[a] + k - 1) * fstride;
      fstride *= m.nf[a];
    }
    out[t] = lin;
  }
}

}  // namespace

void launch_projector_map(const MeshDev& m, unsigned from_mask, unsigned to_mask, long long* out, i64 count,
                          cudaStream_t s) {
  const i64 nb = std::min<i64>((count + 255) / 256, 8 * kNumSms);
  projector_map_kernel<<<static_cast<unsigned>(std::max<i64>(nb, 1)), 256, 0, s>>>(m, from_mask, to_mask, out, count);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_hole_map(const MeshDev& m, long long* out, i64 count, cudaStream_t s) {
  const i64 nb = std::min<i64>((count + 255) / 256, 8 * kNumSms);
  hole_map_kernel<<<static_cast<unsigned>(std::max<i64>(nb, 1)), 256, 0, s>>>(m, out, count);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
