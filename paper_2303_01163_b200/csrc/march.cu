// Fine-grid stencil passes as marching kernels (north-star kernels 1 and 4):
//   RESIDUAL : r = b - A u                                         (fdm.cpp:221-230)
//   UPDATE   : u' = u + s e ; r' = b - A u'                        (solver.cpp:634-645)
//   DOTS     : w = A e ; <r, w>, <w, w>                            (solver.cpp:456-461)
// plus the norms (res_l2, res_inf, err) as block partials folded into the control op.
// Each CTA owns an x-tile and marches along the slowest axis; every value of u/e/b is loaded
// once (x/y neighbours from a double-buffered shared row/plane, the marching-axis neighbours
// from registers), so the pass streams its arrays at HBM speed.  The row sum keeps the
// reference's CSR column order (fdm.cpp:110-117) with non-contracted arithmetic, so r and w
// are bitwise the reference's.
#include "ctrl.cuh"
#include "march.cuh"

#include <algorithm>
#include <cstdlib>

namespace asdsm_b200 {

namespace {

constexpr int TX2 = 128;                      // 2D: threads per x-tile (rows per strip: MarchArgs::strip)
constexpr int TX3 = 32, TY3 = 16;             // 3D: x-by-y tile (z chunk: MarchArgs::strip)

// L2 prefetch of one address (no register is tied up waiting for it)
__device__ __forceinline__ void prefetch_l2(const void* p) { asm volatile("prefetch.global.L2 [%0];" ::"l"(p)); }

// 2D persistent stencil pass: prefetch the next tile's streamed arrays into L2 while this tile
// computes (measured, config 2: update pass 309 -> 252 us with 8-row tiles; the same in the 3D
// z-coarsened pass measured slower at configs 3/4, so it is 2D only; ASDSM_NO_TILE_PREFETCH=1
// turns it off)
template <int MODE>
struct Src {
  const double* __restrict__ u;
  const double* __restrict__ e;
  double s;
  __device__ __forceinline__ double operator()(i64 q) const {
    if (MODE == kMarchUpdate) return __dadd_rn(__ldg(u + q), __dmul_rn(s, __ldg(e + q)));
    if (MODE == kMarchDots) return __ldg(e + q);
    return __ldg(u + q);
  }
};

template <int MODE, bool VAR>
__global__ void __launch_bounds__(TX3 * TY3) march3d_kernel(MarchArgs A) {
  DevState* S = A.state;
  if (!S->active) return;
  const int cur = S->cur;
  double s = 0.0;
  bool work = true;
  if (MODE == kMarchUpdate) {
    s = S->s;
    work = s != 0.0 && (!A.retry_pass || S->retry);
  }
  if (MODE == kMarchDots) work = S->have_e != 0;
  const int Nx = A.g.ext[0], Ny = A.g.ext[1], Nz = A.g.ext[2];
  const i64 sy = A.g.stride[1], sz = A.g.stride[2];
  const Stencil& st = A.st;
  const double* __restrict__ uu = cur ? A.u1 : A.u0;
  const double* __restrict__ ee = A.e;
  Src<MODE> V{uu, ee, s};
  const double* __restrict__ rcur = cur ? A.r1 : A.r0;
  double* __restrict__ uo = MODE == kMarchUpdate ? (cur ? A.uo0 : A.uo1) : nullptr;
  double* __restrict__ ro = MODE == kMarchUpdate ? (cur ? A.ro0 : A.ro1) : (cur ? A.ro1 : A.ro0);
  __shared__ double pl[2][TY3 + 2][TX3 + 2];
  const int SZ = A.strip;
  const int ntx = (Nx + TX3 - 1) / TX3, nty = (Ny + TY3 - 1) / TY3;
  int b = blockIdx.x;
  const int bx = b % ntx;
  b /= ntx;
  const int by = b % nty;
  const int bz = b / nty;
  const int x0 = bx * TX3, y0 = by * TY3, z0 = bz * SZ;
  const int z1 = min(z0 + SZ, Nz);
  const int tx = threadIdx.x % TX3, ty = threadIdx.x / TX3;
  const int x = x0 + tx, y = y0 + ty;
  const bool in = x < Nx && y < Ny;
  // halo roles (each edge thread owns at most one x- and one y-halo cell)
  const bool hxl = in && tx == 0 && x > 0;
  const bool hxr = in && (tx == TX3 - 1 || x == Nx - 1) && x + 1 < Nx;
  const bool hyl = in && ty == 0 && y > 0;
  const bool hyr = in && (ty == TY3 - 1 || y == Ny - 1) && y + 1 < Ny;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (work) {
    const i64 pxy = x + y * sy;
    double vd = (in && z0 > 0) ? V(pxy + (z0 - 1) * sz) : 0.0;
    double vc = in ? V(pxy + z0 * sz) : 0.0;
    double vu = (in && z0 + 1 < Nz) ? V(pxy + (z0 + 1) * sz) : 0.0;
    const i64 p0 = pxy + z0 * sz;
    double hXL = hxl ? V(p0 - 1) : 0.0, hXR = hxr ? V(p0 + 1) : 0.0;
    double hYL = hyl ? V(p0 - sy) : 0.0, hYR = hyr ? V(p0 + sy) : 0.0;
    double bq = (in && MODE != kMarchDots) ? __ldg(A.b + p0) : 0.0;
    double rq = (in && MODE == kMarchDots) ? __ldg(rcur + p0) : 0.0;
    double xq = (in && A.exact && MODE != kMarchDots) ? __ldg(A.exact + p0) : 0.0;
    int buf = 0;
    for (int z = z0; z < z1; ++z) {
      const i64 p = pxy + z * sz;
      double pu = 0.0, pe = 0.0, nXL = 0.0, nXR = 0.0, nYL = 0.0, nYR = 0.0, nb = 0.0, nr = 0.0, nx = 0.0;
      if (in && z + 2 < Nz) {
        pu = (MODE == kMarchDots) ? 0.0 : __ldg(uu + p + 2 * sz);
        if (MODE != kMarchResidual) pe = __ldg(ee + p + 2 * sz);
      }
      if (z + 1 < z1) {
        const i64 pn = p + sz;
        if (hxl) nXL = V(pn - 1);
        if (hxr) nXR = V(pn + 1);
        if (hyl) nYL = V(pn - sy);
        if (hyr) nYR = V(pn + sy);
        if (in && MODE != kMarchDots) nb = __ldg(A.b + pn);
        if (in && MODE == kMarchDots) nr = __ldg(rcur + pn);
        if (in && A.exact && MODE != kMarchDots) nx = __ldg(A.exact + pn);
      }
      pl[buf][ty + 1][tx + 1] = vc;
      if (tx == 0) pl[buf][ty + 1][0] = hXL;
      if (tx == TX3 - 1 || x == Nx - 1) pl[buf][ty + 1][tx + 2] = hXR;
      if (ty == 0) pl[buf][0][tx + 1] = hYL;
      if (ty == TY3 - 1 || y == Ny - 1) pl[buf][ty + 2][tx + 1] = hYR;
      __syncthreads();
      if (in) {
        const i64 N = A.g.size;
        auto C = [&](int slot, double cst) { return VAR ? __ldg(A.coef + slot * N + p) : cst; };
        double acc = 0.0;
        if (z > 0) acc = __dadd_rn(acc, __dmul_rn(C(0, st.left[2]), vd));
        if (y > 0) acc = __dadd_rn(acc, __dmul_rn(C(1, st.left[1]), pl[buf][ty][tx + 1]));
        if (x > 0) acc = __dadd_rn(acc, __dmul_rn(C(2, st.left[0]), pl[buf][ty + 1][tx]));
        acc = __dadd_rn(acc, __dmul_rn(C(3, st.diag), vc));
        if (x < Nx - 1 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(C(4, st.right[0]), pl[buf][ty + 1][tx + 2]));
        if (y < Ny - 1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(C(5, st.right[1]), pl[buf][ty + 2][tx + 1]));
        if (z < Nz - 1 && st.has_right[2]) acc = __dadd_rn(acc, __dmul_rn(C(6, st.right[2]), vu));
        if (MODE == kMarchDots) {
          a0 += rq * acc;
          a2 += acc * acc;
        } else {
          double r = __dsub_rn(bq, acc);
          if (MODE == kMarchUpdate && A.sparse && (x + 1) % A.n[0] != 0 && (y + 1) % A.n[1] != 0 && (z + 1) % A.n[2] != 0)
            r = 0.0;
          ro[p] = r;
          if (MODE == kMarchUpdate) uo[p] = vc;
          a0 += r * r;
          a1 = fmax(a1, fabs(r));
          if (A.exact) {
            const double d = vc - xq;
            a2 += d * d;
            a3 = fmax(a3, fabs(d));
          }
        }
      }
      vd = vc;
      vc = vu;
      if (MODE == kMarchUpdate) vu = __dadd_rn(pu, __dmul_rn(s, pe));
      else if (MODE == kMarchDots) vu = pe;
      else vu = pu;
      hXL = nXL;
      hXR = nXR;
      hYL = nYL;
      hYR = nYR;
      bq = nb;
      rq = nr;
      xq = nx;
      buf ^= 1;
    }
  }
  block_reduce4_march(a0, a1, a2, a3, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}

// Barrier-free 2D variant: 32 x 8 threads over (32 x 8*YC) tiles; each thread owns YC
// consecutive rows of one column and keeps the y-neighbours in registers (YC+2 loads for YC
// points); x-neighbours come through L1 (the adjacent lanes' lines).  No shared memory and no
// per-row barrier: every load of a thread is independent, so the pass is one deep wave of
// loads -- the right shape when the arrays sit in L2 (config 1) and at HBM scale alike.
template <int MODE, bool VAR, int YC>
__device__ __forceinline__ void yc_body(const MarchArgs& A) {
  DevState* S = A.state;
  // state read through volatile: in the fused dots + update kernel it was written by another
  // CTA of the same launch (after the grid barrier)
  const volatile DevState* VS = S;
  if (!VS->active) return;
  const int cur = VS->cur;
  double s = 0.0;
  bool work = true;
  if (MODE == kMarchUpdate) {
    s = VS->s;
    work = s != 0.0 && (!A.retry_pass || VS->retry);
  }
  if (MODE == kMarchDots) work = VS->have_e != 0;
  const int Nx = A.g.ext[0], Ny = A.g.ext[1];
  const i64 sy = A.g.stride[1];
  const Stencil& st = A.st;
  const double* __restrict__ uu = cur ? A.u1 : A.u0;
  Src<MODE> V{uu, A.e, s};
  const double* __restrict__ rcur = cur ? A.r1 : A.r0;
  double* __restrict__ uo = MODE == kMarchUpdate ? (cur ? A.uo0 : A.uo1) : nullptr;
  double* __restrict__ ro = MODE == kMarchUpdate ? (cur ? A.ro0 : A.ro1) : (cur ? A.ro1 : A.ro0);
  double* __restrict__ sta = MODE == kMarchUpdate ? (cur ? A.sta0 : A.sta1) : (cur ? A.sta1 : A.sta0);
  const int ntx = (Nx + 31) / 32, nty = (Ny + 8 * YC - 1) / (8 * YC);
  const int ntiles = ntx * nty;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (int tile = work ? static_cast<int>(blockIdx.x) : ntiles; tile < ntiles; tile += gridDim.x) {
    const int bx = tile % ntx, by = tile / ntx;
    const int x = bx * 32 + tx, y0 = (by * 8 + ty) * YC;
    if (A.prefetch && tile + A.prefetch * static_cast<int>(gridDim.x) < ntiles) {
      const int nt = tile + A.prefetch * gridDim.x;
      const int nx = (nt % ntx) * 32 + tx, ny0 = ((nt / ntx) * 8 + ty) * YC;
      if (nx < Nx)
#pragma unroll
        for (int q = 0; q < YC; ++q) {
          const int y = ny0 + q;
          if (y >= Ny) break;
          const i64 pq = nx + y * sy;
          prefetch_l2(uu + pq);
          if (MODE != kMarchResidual) prefetch_l2(A.e + pq);
          if (MODE != kMarchDots) prefetch_l2(A.b + pq);
          if (MODE == kMarchDots) prefetch_l2(rcur + pq);
          if (A.exact && MODE != kMarchDots) prefetch_l2(A.exact + pq);
        }
    }
    if (x >= Nx || y0 >= Ny) continue;
    // slab-station copies (2D fast path): the column's x-station index, and the row remainder
    // of y0 + 1 modulo n1 advanced incrementally (no divisions in the row loop)
    int xst = -1, yrem = 0;
    if (sta) {
      if ((x + 1) % A.n[0] == 0 && (x + 1) / A.n[0] <= A.nc[0]) xst = (x + 1) / A.n[0] - 1;
      yrem = (y0 + 1) % A.n[1];
    }
    double vy[YC + 2];
#pragma unroll
    for (int q = 0; q < YC + 2; ++q) {
      const int y = y0 - 1 + q;
      vy[q] = (y >= 0 && y < Ny) ? V(x + y * sy) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < YC; ++q) {
      const int y = y0 + q;
      if (y >= Ny) break;
      const i64 p = x + y * sy;
      const i64 N = A.g.size;
      auto C = [&](int slot, double cst) { return VAR ? __ldg(A.coef + slot * N + p) : cst; };
      double acc = 0.0;
      if (y > 0) acc = __dadd_rn(acc, __dmul_rn(C(0, st.left[1]), vy[q]));
      if (x > 0) acc = __dadd_rn(acc, __dmul_rn(C(1, st.left[0]), V(p - 1)));
      const double vc = vy[q + 1];
      acc = __dadd_rn(acc, __dmul_rn(C(2, st.diag), vc));
      if (x < Nx - 1 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(C(3, st.right[0]), V(p + 1)));
      if (y < Ny - 1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(C(4, st.right[1]), vy[q + 2]));
      if (MODE == kMarchDots) {
        const double rp = __ldg(rcur + p);
        a0 += rp * acc;
        a2 += acc * acc;
      } else {
        double r = __dsub_rn(__ldg(A.b + p), acc);
        if (MODE == kMarchUpdate && A.sparse && (x + 1) % A.n[0] != 0 && (y + 1) % A.n[1] != 0) r = 0.0;
        ro[p] = r;
        if (MODE == kMarchUpdate) uo[p] = vc;
        if (sta) {
          if (xst >= 0) sta[static_cast<i64>(xst) * Ny + y] = r;
          if (yrem == 0 && (y + 1) / A.n[1] <= A.nc[1])
            sta[static_cast<i64>(A.nc[0]) * Ny + static_cast<i64>((y + 1) / A.n[1] - 1) * Nx + x] = r;
          yrem = yrem + 1 == A.n[1] ? 0 : yrem + 1;
        }
        a0 += r * r;
        a1 = fmax(a1, fabs(r));
        if (A.exact) {
          const double d = vc - __ldg(A.exact + p);
          a2 += d * d;
          a3 = fmax(a3, fabs(d));
        }
      }
    }
  }
  block_reduce4_march(a0, a1, a2, a3, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}

template <int MODE, bool VAR, int YC>
__global__ void __launch_bounds__(256) stencil2d_yc_kernel(MarchArgs A) {
  pdl_launch_dependents();
  pdl_wait();
  yc_body<MODE, VAR, YC>(A);
}

// A e on the skeleton rows of a 2D mesh (rows at the y-stations, columns at the x-stations,
// each point once), accumulated into <r, Ae> (a0) and <Ae, Ae> (a2) over a grid-stride loop
template <bool VAR>
__device__ __forceinline__ void skel2d_dots_points(const MarchArgs& A, const DevState* S, bool work, double& a0,
                                                   double& a2, unsigned nblk) {
  const int Nx = A.g.ext[0], Ny = A.g.ext[1];
  const i64 sy = A.g.stride[1];
  const Stencil& st = A.st;
  const double* __restrict__ ee = A.e;
  const double* __restrict__ rcur = S->cur ? A.r1 : A.r0;
  const int nc0 = A.nc[0], nc1 = A.nc[1], n0 = A.n[0], n1 = A.n[1];
  const i64 nrow = static_cast<i64>(nc1) * Nx, ncol = static_cast<i64>(nc0) * Ny;
  for (i64 t = work ? static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x : nrow + ncol; t < nrow + ncol;
       t += static_cast<i64>(nblk) * blockDim.x) {
    int x, y;
    if (t < nrow) {
      const int J = static_cast<int>(t / Nx);
      x = static_cast<int>(t - static_cast<i64>(J) * Nx);
      y = (J + 1) * n1 - 1;
    } else {
      const i64 tc = t - nrow;
      const int I = static_cast<int>(tc / Ny);
      y = static_cast<int>(tc - static_cast<i64>(I) * Ny);
      if ((y + 1) % n1 == 0) continue;  // cross point: counted with the rows
      x = (I + 1) * n0 - 1;
    }
    const i64 p = x + y * sy;
    const i64 N = A.g.size;
    auto C = [&](int slot, double cst) { return VAR ? __ldg(A.coef + slot * N + p) : cst; };
    double acc = 0.0;
    if (y > 0) acc = __dadd_rn(acc, __dmul_rn(C(0, st.left[1]), __ldg(ee + p - sy)));
    if (x > 0) acc = __dadd_rn(acc, __dmul_rn(C(1, st.left[0]), __ldg(ee + p - 1)));
    acc = __dadd_rn(acc, __dmul_rn(C(2, st.diag), __ldg(ee + p)));
    if (x < Nx - 1 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(C(3, st.right[0]), __ldg(ee + p + 1)));
    if (y < Ny - 1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(C(4, st.right[1]), __ldg(ee + p + sy)));
    a0 += __ldg(rcur + p) * acc;
    a2 += acc * acc;
  }
}

// Skeleton-row step dots and the update in one launch.  Phase 1 is skel2d_dots_kernel's work;
// its last block applies the step control and bumps DevState::gen; every CTA waits for the bump
// (the grid is co-resident: cooperative launch, occupancy checked on the host; the wait is
// bounded and traps rather than hang), then runs the update pass with the new step.  One
// launch, one grid barrier, instead of two kernels with a launch boundary between them.
template <int YC>
__global__ void __launch_bounds__(256, 4) dots_update2d_kernel(MarchArgs A) {
  DevState* S = A.state;
  if (!S->active) return;
  unsigned gen0;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(gen0) : "l"(&S->gen) : "memory");
  // phase 1 on the first blocks only (one skeleton point per thread): fewer arrivals and
  // partials for the last block to fold; the other blocks go straight to the barrier
  const i64 npts = static_cast<i64>(A.nc[1]) * A.g.ext[0] + static_cast<i64>(A.nc[0]) * A.g.ext[1];
  const unsigned nd = static_cast<unsigned>(((npts + blockDim.x - 1) / blockDim.x < static_cast<i64>(gridDim.x) ? (npts + blockDim.x - 1) / blockDim.x : static_cast<i64>(gridDim.x)));
  bool released = false;
  if (blockIdx.x < nd) {
    double a0 = 0.0, a2 = 0.0;
    skel2d_dots_points<false>(A, S, S->have_e != 0, a0, a2, nd);
    block_reduce4_march(a0, 0.0, a2, 0.0, A.partials);
    if (fold_ctrl(A.dots_ctrl, A.partials, S, A.history, nd)) {
      released = true;
      if (threadIdx.x == 0) {
        __threadfence();
        asm volatile("red.release.gpu.global.add.u32 [%0], 1;" ::"l"(&S->gen) : "memory");
      }
    }
  }
  if (!released && threadIdx.x == 0) {
    unsigned g, n = 0;
    do {
      asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(g) : "l"(&S->gen) : "memory");
      if (g != gen0) break;
      __nanosleep(128);
      if (++n > (1u << 24)) __trap();  // a grid that is not co-resident: fail, do not hang
    } while (true);
  }
  __syncthreads();
  yc_body<kMarchUpdate, false, YC>(A);
}

// DOTS restricted to the skeleton rows of a 2D mesh (rows at the y-stations, columns at the
// x-stations, each point once): same per-point arithmetic as the full pass.
template <bool VAR>
__global__ void __launch_bounds__(128) skel2d_dots_kernel(MarchArgs A) {
  DevState* S = A.state;
  if (!S->active) return;
  double a0 = 0.0, a2 = 0.0;
  skel2d_dots_points<VAR>(A, S, S->have_e != 0, a0, a2, gridDim.x);
  block_reduce4_march(a0, 0.0, a2, 0.0, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}

// 3D counterpart: the union of the station planes (x-planes, then y-planes off the x-stations,
// then z-planes off both), each point once, same per-point arithmetic as march3d's DOTS.
template <bool VAR>
__global__ void __launch_bounds__(256) skel3d_dots_kernel(MarchArgs A) {
  DevState* S = A.state;
  if (!S->active) return;
  const bool work = S->have_e != 0;
  const int Nx = A.g.ext[0], Ny = A.g.ext[1], Nz = A.g.ext[2];
  const i64 sy = A.g.stride[1], sz = A.g.stride[2];
  const Stencil& st = A.st;
  const double* __restrict__ ee = A.e;
  const double* __restrict__ rcur = S->cur ? A.r1 : A.r0;
  const int n0 = A.n[0], n1 = A.n[1], n2 = A.n[2];
  const i64 px = static_cast<i64>(A.nc[0]) * Ny * Nz;  // x-planes: (I, y, z), y fastest
  const i64 py = static_cast<i64>(A.nc[1]) * Nx * Nz;  // y-planes: (J, x, z), x fastest
  const i64 pz = static_cast<i64>(A.nc[2]) * Nx * Ny;  // z-planes: (K, x, y), x fastest
  double a0 = 0.0, a2 = 0.0;
  for (i64 t = work ? static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x : px + py + pz; t < px + py + pz;
       t += static_cast<i64>(gridDim.x) * blockDim.x) {
    int x, y, z;
    if (t < px) {
      const i64 q = t / Ny;
      y = static_cast<int>(t - q * Ny);
      const int I = static_cast<int>(q / Nz);
      z = static_cast<int>(q - static_cast<i64>(I) * Nz);
      x = (I + 1) * n0 - 1;
    } else if (t < px + py) {
      const i64 u = t - px, q = u / Nx;
      x = static_cast<int>(u - q * Nx);
      if ((x + 1) % n0 == 0) continue;
      const int J = static_cast<int>(q / Nz);
      z = static_cast<int>(q - static_cast<i64>(J) * Nz);
      y = (J + 1) * n1 - 1;
    } else {
      const i64 u = t - px - py, q = u / Nx;
      x = static_cast<int>(u - q * Nx);
      const int K = static_cast<int>(q / Ny);
      y = static_cast<int>(q - static_cast<i64>(K) * Ny);
      if ((x + 1) % n0 == 0 || (y + 1) % n1 == 0) continue;
      z = (K + 1) * n2 - 1;
    }
    const i64 p = x + y * sy + z * sz;
    const i64 N = A.g.size;
    auto C = [&](int slot, double cst) { return VAR ? __ldg(A.coef + slot * N + p) : cst; };
    double acc = 0.0;
    if (z > 0) acc = __dadd_rn(acc, __dmul_rn(C(0, st.left[2]), __ldg(ee + p - sz)));
    if (y > 0) acc = __dadd_rn(acc, __dmul_rn(C(1, st.left[1]), __ldg(ee + p - sy)));
    if (x > 0) acc = __dadd_rn(acc, __dmul_rn(C(2, st.left[0]), __ldg(ee + p - 1)));
    acc = __dadd_rn(acc, __dmul_rn(C(3, st.diag), __ldg(ee + p)));
    if (x < Nx - 1 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(C(4, st.right[0]), __ldg(ee + p + 1)));
    if (y < Ny - 1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(C(5, st.right[1]), __ldg(ee + p + sy)));
    if (z < Nz - 1 && st.has_right[2]) acc = __dadd_rn(acc, __dmul_rn(C(6, st.right[2]), __ldg(ee + p + sz)));
    a0 += __ldg(rcur + p) * acc;
    a2 += acc * acc;
  }
  block_reduce4_march(a0, 0.0, a2, 0.0, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}

// Same sums over the same points, one warp per skeleton row: x-plane rows (I, z) run along y,
// y-plane rows (J, z) and z-plane rows (K, y) along x, so there is no 64-bit division per point
// (the kernel above spends ~6) and each lane has four points' loads in flight at once.
template <bool VAR>
__global__ void __launch_bounds__(256) skel3d_dots_rows_kernel(MarchArgs A) {
  DevState* S = A.state;
  if (!S->active) return;
  const bool work = S->have_e != 0;
  const int Nx = A.g.ext[0], Ny = A.g.ext[1], Nz = A.g.ext[2];
  const i64 sy = A.g.stride[1], sz = A.g.stride[2];
  const Stencil& st = A.st;
  const double* __restrict__ ee = A.e;
  const double* __restrict__ rcur = S->cur ? A.r1 : A.r0;
  const int n0 = A.n[0], n1 = A.n[1], n2 = A.n[2];
  const int rx = A.nc[0] * Nz, ry = A.nc[1] * Nz, rz = A.nc[2] * Ny;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, nw = (gridDim.x * blockDim.x) >> 5;
  double a0 = 0.0, a2 = 0.0;
  for (int row = work ? gw : rx + ry + rz; row < rx + ry + rz; row += nw) {
    int fam, x = 0, y = 0, z = 0, len;
    if (row < rx) {  // (I, z): y varies
      fam = 0;
      z = row % Nz;
      x = (row / Nz + 1) * n0 - 1;
      len = Ny;
    } else if (row < rx + ry) {  // (J, z): x varies
      fam = 1;
      const int q = row - rx;
      z = q % Nz;
      y = (q / Nz + 1) * n1 - 1;
      len = Nx;
    } else {  // (K, y): x varies; rows on a y-station belong to the y-planes
      fam = 2;
      const int q = row - rx - ry;
      y = q % Ny;
      z = (q / Ny + 1) * n2 - 1;
      if ((y + 1) % n1 == 0) continue;
      len = Nx;
    }
    const i64 base = fam == 0 ? x + z * sz : y * sy + z * sz;
    const i64 step = fam == 0 ? sy : 1;
    for (int v0 = lane; v0 < len; v0 += 128) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int v = v0 + 32 * u;
        if (v >= len) break;
        const int px = fam == 0 ? x : v, py = fam == 0 ? v : y;
        if (fam != 0 && (px + 1) % n0 == 0) continue;  // x-station points: counted with the x-planes
        const i64 p = base + v * step;
        const i64 N = A.g.size;
        auto C = [&](int slot, double cst) { return VAR ? __ldg(A.coef + slot * N + p) : cst; };
        double acc = 0.0;
        if (z > 0) acc = __dadd_rn(acc, __dmul_rn(C(0, st.left[2]), __ldg(ee + p - sz)));
        if (py > 0) acc = __dadd_rn(acc, __dmul_rn(C(1, st.left[1]), __ldg(ee + p - sy)));
        if (px > 0) acc = __dadd_rn(acc, __dmul_rn(C(2, st.left[0]), __ldg(ee + p - 1)));
        acc = __dadd_rn(acc, __dmul_rn(C(3, st.diag), __ldg(ee + p)));
        if (px < Nx - 1 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(C(4, st.right[0]), __ldg(ee + p + 1)));
        if (py < Ny - 1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(C(5, st.right[1]), __ldg(ee + p + sy)));
        if (z < Nz - 1 && st.has_right[2]) acc = __dadd_rn(acc, __dmul_rn(C(6, st.right[2]), __ldg(ee + p + sz)));
        a0 += __ldg(rcur + p) * acc;
        a2 += acc * acc;
      }
    }
  }
  block_reduce4_march(a0, 0.0, a2, 0.0, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}

// Barrier-free 3D variant: persistent blocks of 32x8 threads over (32 x 8 x ZC) tiles; each
// thread owns ZC consecutive z points and keeps the z-neighbours in registers (ZC+2 loads for
// ZC points), x/y neighbours come through L1 (same or adjacent warps' lines).
#ifndef ASDSM_ZC
#define ASDSM_ZC 8
#endif
#ifndef ASDSM_ZC_MINB
#define ASDSM_ZC_MINB 4
#endif
constexpr int ZC = ASDSM_ZC;
template <int MODE, bool VAR>
__global__ void __launch_bounds__(256, ASDSM_ZC_MINB) stencil3d_zc_kernel(MarchArgs A) {
  DevState* S = A.state;
  if (!S->active) return;
  const int cur = S->cur;
  double s = 0.0;
  bool work = true;
  if (MODE == kMarchUpdate || MODE == kMarchCand) {
    s = S->s;
    work = s != 0.0 && (!A.retry_pass || S->retry);
  }
  if (MODE == kMarchDots) work = S->have_e != 0;
  const int Nx = A.g.ext[0], Ny = A.g.ext[1], Nz = A.g.ext[2];
  const i64 sy = A.g.stride[1], sz = A.g.stride[2];
  const Stencil& st = A.st;
  const double* __restrict__ uu = MODE == kMarchCand ? (cur ? A.uo0 : A.uo1) : (cur ? A.u1 : A.u0);
  Src<MODE> V{uu, A.e, s};
  const double* __restrict__ rcur = cur ? A.r1 : A.r0;
  double* __restrict__ uo = MODE == kMarchUpdate ? (cur ? A.uo0 : A.uo1) : nullptr;
  double* __restrict__ ro =
      (MODE == kMarchUpdate || MODE == kMarchCand) ? (cur ? A.ro0 : A.ro1) : (cur ? A.ro1 : A.ro0);
  const int ntx = (Nx + 31) / 32, nty = (Ny + 7) / 8, ntz = (Nz + ZC - 1) / ZC;
  const long long ntiles = static_cast<long long>(ntx) * nty * ntz;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  for (long long tile = work ? blockIdx.x : ntiles; tile < ntiles; tile += gridDim.x) {
    const int bx = static_cast<int>(tile % ntx);
    const int by = static_cast<int>((tile / ntx) % nty);
    const int bz = static_cast<int>(tile / (static_cast<long long>(ntx) * nty));
    const int x = bx * 32 + tx, y = by * 8 + ty, z0 = bz * ZC;
    if (x >= Nx || y >= Ny) continue;
    const i64 pxy = x + y * sy;
    double vz[ZC + 2];
#pragma unroll
    for (int q = 0; q < ZC + 2; ++q) {
      const int z = z0 - 1 + q;
      vz[q] = (z >= 0 && z < Nz) ? V(pxy + z * sz) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < ZC; ++q) {
      const int z = z0 + q;
      if (z >= Nz) break;
      const i64 p = pxy + z * sz;
      const i64 N = A.g.size;
      auto C = [&](int slot, double cst) { return VAR ? __ldg(A.coef + slot * N + p) : cst; };
      double acc = 0.0;
      if (z > 0) acc = __dadd_rn(acc, __dmul_rn(C(0, st.left[2]), vz[q]));
      if (y > 0) acc = __dadd_rn(acc, __dmul_rn(C(1, st.left[1]), V(p - sy)));
      if (x > 0) acc = __dadd_rn(acc, __dmul_rn(C(2, st.left[0]), V(p - 1)));
      const double vc = vz[q + 1];
      acc = __dadd_rn(acc, __dmul_rn(C(3, st.diag), vc));
      if (x < Nx - 1 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(C(4, st.right[0]), V(p + 1)));
      if (y < Ny - 1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(C(5, st.right[1]), V(p + sy)));
      if (z < Nz - 1 && st.has_right[2]) acc = __dadd_rn(acc, __dmul_rn(C(6, st.right[2]), vz[q + 2]));
      if (MODE == kMarchDots) {
        const double rp = __ldg(rcur + p);
        a0 += rp * acc;
        a2 += acc * acc;
      } else {
        double r = __dsub_rn(__ldg(A.b + p), acc);
        if ((MODE == kMarchUpdate || MODE == kMarchCand) && A.sparse && (x + 1) % A.n[0] != 0 &&
            (y + 1) % A.n[1] != 0 && (z + 1) % A.n[2] != 0)
          r = 0.0;
        ro[p] = r;
        if (MODE == kMarchUpdate) uo[p] = vc;
        a0 += r * r;
        a1 = fmax(a1, fabs(r));
        if (A.exact) {
          const double d = vc - __ldg(A.exact + p);
          a2 += d * d;
          a3 = fmax(a3, fabs(d));
        }
      }
    }
  }
  block_reduce4_march(a0, a1, a2, a3, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}


// Lean y-march of the 2D constant-coefficient passes (the 2D form of stencil3d_zm_kernel below):
//   RESIDUAL : r = b - A u        UPDATE : v = u + s e ; u' = v ; r' = b - A v ; norms
// plus the residual's copies on the slab stations.  A CTA owns 256 consecutive columns and a row
// range; a thread walks its column in chunks of YM rows: one up-front batch of the chunk's
// next-row values and b (exact) values, the two trailing rows carried in registers, x neighbours
// from L1.  The row index is CTA-uniform, so the y-station test is a uniform branch; domain edges
// are clamped neighbour offsets with zeroed per-thread coefficients (adding c * v = +-0 to a
// row sum that starts at +0 leaves it bitwise unchanged).  32-bit indices (size < 2^31).
constexpr int YM = 4;
template <int MODE, bool EX>
__global__ void __launch_bounds__(256, (MODE == kMarchUpdate && EX) ? 3 : 4) stencil2d_ym_kernel(MarchArgs A, int ylen) {
  pdl_launch_dependents();
  pdl_wait();
  DevState* S = A.state;
  if (!S->active) return;
  const int cur = S->cur;
  double sc = 0.0;
  bool work = true;
  if (MODE == kMarchUpdate) {
    sc = S->s;
    work = sc != 0.0 && (!A.retry_pass || S->retry);
  }
  const int Nx = A.g.ext[0], Ny = A.g.ext[1];
  const int sy = Nx;
  const Stencil& st = A.st;
  const double* __restrict__ uu = cur ? A.u1 : A.u0;
  const double* __restrict__ ee = A.e;
  const double* __restrict__ bb = A.b;
  const double* __restrict__ xx = A.exact;
  double* __restrict__ uo = MODE == kMarchUpdate ? (cur ? A.uo0 : A.uo1) : nullptr;
  double* __restrict__ rr = MODE == kMarchUpdate ? (cur ? A.ro0 : A.ro1) : (cur ? A.ro1 : A.ro0);
  double* __restrict__ sta = MODE == kMarchUpdate ? (cur ? A.sta0 : A.sta1) : (cur ? A.sta1 : A.sta0);
  const unsigned ntx = (Nx + 255) / 256;
  const unsigned bx = blockIdx.x % ntx, byr = blockIdx.x / ntx;
  const int x0 = bx * 256 + threadIdx.x;
  const bool in = x0 < Nx;
  const int x = min(x0, Nx - 1);
  const int oxl = x > 0 ? -1 : 0, oxr = x < Nx - 1 ? 1 : 0;
  const double cxl = x > 0 ? st.left[0] : 0.0, cxr = (x < Nx - 1 && st.has_right[0]) ? st.right[0] : 0.0;
  const double cyr = st.has_right[1] ? st.right[1] : 0.0;
  const int yb = byr * ylen, ye = work ? min(Ny, yb + ylen) : yb;
  int i = x + yb * sy;
  // station copies: this column's x-station slot (or -1); the y-station test is per row, uniform
  int xst = -1;
  if (sta && in && (x + 1) % A.n[0] == 0 && (x + 1) / A.n[0] <= A.nc[0]) xst = ((x + 1) / A.n[0] - 1) * Ny;
  int yrem = (yb + 1) % A.n[1], yJ = (yb + 1) / A.n[1];
  auto V = [&](int j) -> double {
    if (MODE == kMarchUpdate) return __dadd_rn(__ldg(uu + j), __dmul_rn(sc, __ldg(ee + j)));
    return __ldg(uu + j);
  };
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  double vm = 0.0, vc = 0.0;
  if (yb < ye) {
    vm = yb > 0 ? V(i - sy) : 0.0;
    vc = V(i);
  }
  for (int y0 = yb; y0 < ye; y0 += YM) {
    double vn[YM], bq[YM], eq[EX ? YM : 1];
#pragma unroll
    for (int q = 0; q < YM; ++q) {
      const int y = y0 + q;
      const int j = i + q * sy;
      vn[q] = y + 1 < Ny ? V(j + sy) : 0.0;
      bq[q] = y < Ny ? __ldg(bb + j) : 0.0;
      if (EX) eq[q] = y < Ny ? __ldg(xx + j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < YM; ++q) {
      const int y = y0 + q;
      if (y < ye) {
        const int j = i + q * sy;
        double acc = __dadd_rn(0.0, __dmul_rn(y > 0 ? st.left[1] : 0.0, vm));
        acc = __dadd_rn(acc, __dmul_rn(cxl, V(j + oxl)));
        acc = __dadd_rn(acc, __dmul_rn(st.diag, vc));
        acc = __dadd_rn(acc, __dmul_rn(cxr, V(j + oxr)));
        acc = __dadd_rn(acc, __dmul_rn(y < Ny - 1 ? cyr : 0.0, vn[q]));
        const double r = __dsub_rn(bq[q], acc);
        if (in) {
          rr[j] = r;
          if (MODE == kMarchUpdate) uo[j] = vc;
          if (xst >= 0) sta[xst + y] = r;
          if (sta && yrem == 0 && yJ <= A.nc[1]) sta[A.nc[0] * Ny + (yJ - 1) * Nx + x] = r;
          a0 += r * r;
          a1 = fmax(a1, fabs(r));
          if (EX) {
            const double d = vc - eq[q];
            a2 += d * d;
            a3 = fmax(a3, fabs(d));
          }
        }
        if (++yrem == A.n[1]) {
          yrem = 0;
          ++yJ;
        }
        vm = vc;
        vc = vn[q];
      }
    }
    i += YM * sy;
  }
  block_reduce4_march(a0, a1, a2, a3, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}

static bool ym_supported(const MarchArgs& A) {
  const FineGeom& g = A.g;
  return g.dim == 2 && A.coef == nullptr && !A.sparse && g.size < (1LL << 31) - (1LL << 20) && g.stride[1] == g.ext[0] &&
         (!A.sta0 || static_cast<long long>(A.nc[0]) * g.ext[1] + static_cast<long long>(A.nc[1]) * g.ext[0] < (1LL << 31));
}

// row-range length: ~8 CTAs per SM over the whole grid, whole chunks, at least four chunks
// (measured at config 1: ranges of 8 / 16 / 32 rows 1.160 / 1.134 / 1.232 ms per solve)
static int ym_ylen(const FineGeom& g) {
  if (const char* e = std::getenv("ASDSM_YM_LEN")) return std::max(YM, std::atoi(e) / YM * YM);
  const int ntx = (g.ext[0] + 255) / 256;
  const int nyr = std::max(1, 8 * kNumSms / ntx);
  int ylen = ((g.ext[1] + nyr - 1) / nyr + YM - 1) / YM * YM;
  ylen = std::max(ylen, 4 * YM);
  while (static_cast<long long>(ntx) * ((g.ext[1] + ylen - 1) / ylen) > kRedStride) ylen += YM;
  return ylen;
}

template <int MODE>
static void launch_ym(const MarchArgs& A, cudaStream_t s) {
  const int ylen = ym_ylen(A.g);
  const unsigned nb = static_cast<unsigned>(((A.g.ext[0] + 255) / 256) * ((A.g.ext[1] + ylen - 1) / ylen));
  if (A.exact) launch_pdl(stencil2d_ym_kernel<MODE, true>, nb, 256, 0, s, A, ylen);
  else launch_pdl(stencil2d_ym_kernel<MODE, false>, nb, 256, 0, s, A, ylen);
}

// Lean z-march of the 3D constant-coefficient passes (north-star kernels 1 and 4 in 3D):
//   RESIDUAL : r = b - A u            CAND : r' = b - A u' (u' from the axpy pass)
//   UPDATE   : v = u + s e ; u' = v ; r' = b - A v   (solver.cpp:634-645, fdm.cpp:221-230)
// A CTA of 32 x 8 threads owns one xy tile and a z range; a thread walks its column in chunks
// of ZM planes: one up-front batch of the chunk's next-plane values and b (exact) values, the two
// trailing planes carried in registers (no z halo re-read), in-plane neighbours from L1 (lines
// the neighbouring warps' batches fetched).  Measured against the tile-walking z-coarsened
// kernel (scripts/probe_stencil3d.cu, 509^3): that kernel issues ~115 instructions per point --
// three 64-bit divisions per tile, 64-bit addresses, per-point boundary predicates -- and is
// issue/latency bound at 3.8 TB/s with DRAM traffic already at the algorithmic bytes; here the
// tile is fixed per CTA (32-bit division once), indices are 32-bit (size < 2^31), and the domain
// edges are clamped neighbour offsets with zeroed per-thread coefficients: c * v = +-0 added to
// a row sum that starts at +0 and therefore is never -0 leaves it bitwise unchanged, so r is
// bitwise the reference's CSR row sum (fdm.cpp:110-117) as before.
constexpr int ZM = 4;
template <int MODE, bool EX>
__global__ void __launch_bounds__(256, (MODE == kMarchUpdate && EX) ? 3 : 4) stencil3d_zm_kernel(MarchArgs A, int zlen) {
  DevState* S = A.state;
  if (!S->active) return;
  const int cur = S->cur;
  double sc = 0.0;
  bool work = true;
  if (MODE == kMarchUpdate || MODE == kMarchCand) {
    sc = S->s;
    work = sc != 0.0 && (!A.retry_pass || S->retry);
  }
  const int Nx = A.g.ext[0], Ny = A.g.ext[1], Nz = A.g.ext[2];
  const int sy = Nx, sz = Nx * Ny;
  const Stencil& st = A.st;
  const double* __restrict__ uu = MODE == kMarchCand ? (cur ? A.uo0 : A.uo1) : (cur ? A.u1 : A.u0);
  const double* __restrict__ ee = A.e;
  const double* __restrict__ bb = A.b;
  const double* __restrict__ xx = A.exact;
  double* __restrict__ uo = MODE == kMarchUpdate ? (cur ? A.uo0 : A.uo1) : nullptr;
  double* __restrict__ rr = MODE == kMarchResidual ? (cur ? A.ro1 : A.ro0) : (cur ? A.ro0 : A.ro1);
  const unsigned ntx = (Nx + 31) / 32, nty = (Ny + 7) / 8;
  unsigned t = blockIdx.x;
  const unsigned bx = t % ntx;
  t /= ntx;
  const unsigned by = t % nty, bzr = t / nty;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  const int x0 = bx * 32 + tx, y0 = by * 8 + ty;
  const bool in = x0 < Nx && y0 < Ny;
  const int x = min(x0, Nx - 1), y = min(y0, Ny - 1);
  const int oxl = x > 0 ? -1 : 0, oxr = x < Nx - 1 ? 1 : 0, oyl = y > 0 ? -sy : 0, oyr = y < Ny - 1 ? sy : 0;
  const double cxl = x > 0 ? st.left[0] : 0.0, cxr = (x < Nx - 1 && st.has_right[0]) ? st.right[0] : 0.0;
  const double cyl = y > 0 ? st.left[1] : 0.0, cyr = (y < Ny - 1 && st.has_right[1]) ? st.right[1] : 0.0;
  const double czr = st.has_right[2] ? st.right[2] : 0.0;
  const int zb = bzr * zlen, ze = work ? min(Nz, zb + zlen) : zb;
  int i = x + y * sy + zb * sz;  // element index of (x, y, zb)
  auto V = [&](int j) -> double {
    if (MODE == kMarchUpdate) return __dadd_rn(__ldg(uu + j), __dmul_rn(sc, __ldg(ee + j)));
    return __ldg(uu + j);
  };
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  double vm = 0.0, vc = 0.0;
  if (zb < ze) {
    vm = zb > 0 ? V(i - sz) : 0.0;  // plane z - 1
    vc = V(i);                       // plane z
  }
  for (int z0 = zb; z0 < ze; z0 += ZM) {
    double vn[ZM], bq[ZM], eq[EX ? ZM : 1];
#pragma unroll
    for (int q = 0; q < ZM; ++q) {
      const int z = z0 + q;
      const int j = i + q * sz;
      vn[q] = z + 1 < Nz ? V(j + sz) : 0.0;
      bq[q] = z < Nz ? __ldg(bb + j) : 0.0;
      if (EX) eq[q] = z < Nz ? __ldg(xx + j) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < ZM; ++q) {
      const int z = z0 + q;
      if (z < ze) {
        const int j = i + q * sz;
        double acc = __dadd_rn(0.0, __dmul_rn(z > 0 ? st.left[2] : 0.0, vm));
        acc = __dadd_rn(acc, __dmul_rn(cyl, V(j + oyl)));
        acc = __dadd_rn(acc, __dmul_rn(cxl, V(j + oxl)));
        acc = __dadd_rn(acc, __dmul_rn(st.diag, vc));
        acc = __dadd_rn(acc, __dmul_rn(cxr, V(j + oxr)));
        acc = __dadd_rn(acc, __dmul_rn(cyr, V(j + oyr)));
        acc = __dadd_rn(acc, __dmul_rn(z < Nz - 1 ? czr : 0.0, vn[q]));
        const double r = __dsub_rn(bq[q], acc);
        if (in) {
          rr[j] = r;
          if (MODE == kMarchUpdate) uo[j] = vc;
          a0 += r * r;
          a1 = fmax(a1, fabs(r));
          if (EX) {
            const double d = vc - eq[q];
            a2 += d * d;
            a3 = fmax(a3, fabs(d));
          }
        }
        vm = vc;
        vc = vn[q];
      }
    }
    i += ZM * sz;
  }
  block_reduce4_march(a0, a1, a2, a3, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}

// z-range length of the lean z-march: ~8 ranges per column (whole chunks), more planes per range
// when the grid would exceed the partial buffer
static int zm_zlen(const FineGeom& g) {
  const long long nxy = static_cast<long long>((g.ext[0] + 31) / 32) * ((g.ext[1] + 7) / 8);
  int zlen = ((g.ext[2] + 7) / 8 + ZM - 1) / ZM * ZM;
  while (nxy * ((g.ext[2] + zlen - 1) / zlen) > kRedStride) zlen += ZM;
  return zlen;
}

static bool zm_supported(const MarchArgs& A) {
  const FineGeom& g = A.g;
  return g.dim == 3 && A.coef == nullptr && !A.sparse && g.size < (1LL << 31) - (1LL << 20) && g.stride[1] == g.ext[0] &&
         g.stride[2] == static_cast<i64>(g.ext[0]) * g.ext[1] &&
         static_cast<long long>((g.ext[0] + 31) / 32) * ((g.ext[1] + 7) / 8) <= kRedStride;
}

template <int MODE>
static void launch_zm(const MarchArgs& A, cudaStream_t s) {
  const int zlen = zm_zlen(A.g);
  const unsigned nb = static_cast<unsigned>(((A.g.ext[0] + 31) / 32) * ((A.g.ext[1] + 7) / 8) * ((A.g.ext[2] + zlen - 1) / zlen));
  if (A.exact) stencil3d_zm_kernel<MODE, true><<<nb, 256, 0, s>>>(A, zlen);
  else stencil3d_zm_kernel<MODE, false><<<nb, 256, 0, s>>>(A, zlen);
}

// The 3D update's first pass: u' = u + s e into the non-current buffer (vectorized stream);
// the residual of u' follows as kMarchCand (measured: two passes stream faster than the fused
// 3D update, whose neighbour values each cost two loads).
__global__ void __launch_bounds__(256) axpy_update_kernel(MarchArgs A) {
  const DevState* S = A.state;
  if (!S->active) return;
  const double s = S->s;
  if (!(s != 0.0 && (!A.retry_pass || S->retry))) return;
  const int cur = S->cur;
  const double* __restrict__ u = cur ? A.u1 : A.u0;
  const double* __restrict__ e = A.e;
  double* __restrict__ uo = cur ? A.uo0 : A.uo1;
  const i64 n = A.g.size, n2 = n / 2;
  const i64 stride = static_cast<i64>(gridDim.x) * blockDim.x;
  for (i64 i = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; i < n2; i += stride) {
    const double2 uv = __ldg(reinterpret_cast<const double2*>(u) + i);
    const double2 ev = __ldg(reinterpret_cast<const double2*>(e) + i);
    reinterpret_cast<double2*>(uo)[i] = make_double2(__dadd_rn(uv.x, __dmul_rn(s, ev.x)), __dadd_rn(uv.y, __dmul_rn(s, ev.y)));
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (n & 1)) uo[n - 1] = __dadd_rn(u[n - 1], __dmul_rn(s, e[n - 1]));
}
}  // namespace

int march_strip(const FineGeom& g) {
  // enough CTAs to cover 148 SMs several times, strips of 4..32 rows (planes in 3D)
  if (g.dim == 3) {
    const long long nt = ((g.ext[0] + TX3 - 1) / TX3) * ((g.ext[1] + TY3 - 1) / TY3);
    long long sz = (static_cast<long long>(g.ext[2]) * nt) / (4LL * kNumSms);
    if (sz < 4) sz = 4;
    if (sz > 64) sz = 64;
    return static_cast<int>(sz);
  }
  const long long ntx = (g.ext[0] + TX2 - 1) / TX2;
  long long sy = (static_cast<long long>(g.ext[1]) * ntx) / (8LL * kNumSms);
  if (sy < 4) sy = 4;
  if (sy > 32) sy = 32;
  return static_cast<int>(sy);
}

unsigned march_blocks(const FineGeom& g) {
  if (g.dim == 2) {
    const int sy = march_strip(g);
    return static_cast<unsigned>(((g.ext[0] + TX2 - 1) / TX2) * ((g.ext[1] + sy - 1) / sy));
  }
  const int sz = march_strip(g);
  return static_cast<unsigned>(((g.ext[0] + TX3 - 1) / TX3) * ((g.ext[1] + TY3 - 1) / TY3) * ((g.ext[2] + sz - 1) / sz));
}

static unsigned dots_update_blocks(const FineGeom& g) {
  constexpr int kYc = 8;
  const long long tiles = static_cast<long long>((g.ext[0] + 31) / 32) * ((g.ext[1] + 8 * kYc - 1) / (8 * kYc));
  return static_cast<unsigned>(std::min<long long>(tiles, 4LL * kNumSms));
}

bool dots_update_supported(const FineGeom& g) {
  static int resident = -1;
  if (resident < 0) {
    int dev = 0, sms = 0, per_sm = 0;
    ASDSM_CUDA_CHECK(cudaGetDevice(&dev));
    ASDSM_CUDA_CHECK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    ASDSM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, dots_update2d_kernel<8>, 256, 0));
    resident = sms * per_sm;
  }
  return g.dim == 2 && static_cast<long long>(dots_update_blocks(g)) <= resident;
}

void launch_march(int mode, const MarchArgs& A0, cudaStream_t s) {
  MarchArgs A = A0;
  const bool no_prefetch = std::getenv("ASDSM_NO_TILE_PREFETCH") != nullptr;
  const int dist = std::getenv("ASDSM_PREFETCH_DIST") ? std::atoi(std::getenv("ASDSM_PREFETCH_DIST")) : 1;
  A.prefetch = no_prefetch ? 0 : dist;
  A.strip = march_strip(A.g);
  const unsigned nb = march_blocks(A.g);
  if (nb > static_cast<unsigned>(kRedStride)) throw AsdsmError(kUnsupported, "fine grid too large for the partial buffer");
  const bool var = A.coef != nullptr;
#define ASDSM_MARCH_DISPATCH(KERNEL, GRID, BLOCK)                                        \
  do {                                                                                  \
    if (var) {                                                                          \
      if (mode == kMarchResidual) KERNEL<kMarchResidual, true><<<GRID, BLOCK, 0, s>>>(A); \
      else if (mode == kMarchUpdate) KERNEL<kMarchUpdate, true><<<GRID, BLOCK, 0, s>>>(A); \
      else KERNEL<kMarchDots, true><<<GRID, BLOCK, 0, s>>>(A);                         \
    } else {                                                                            \
      if (mode == kMarchResidual) KERNEL<kMarchResidual, false><<<GRID, BLOCK, 0, s>>>(A); \
      else if (mode == kMarchUpdate) KERNEL<kMarchUpdate, false><<<GRID, BLOCK, 0, s>>>(A); \
      else KERNEL<kMarchDots, false><<<GRID, BLOCK, 0, s>>>(A);                        \
    }                                                                                   \
  } while (0)
  if (mode == kMarchDotsUpdate) {
    if (A.g.dim != 2 || var || !A.skel_only) throw AsdsmError(kUnsupported, "fused dots + update: 2D constant coefficients");
    constexpr int kYc = 8;
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(dots_update_blocks(A.g));
    cfg.blockDim = dim3(256);
    cfg.stream = s;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeCooperative;
    attr[0].val.cooperative = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    ASDSM_CUDA_CHECK(cudaLaunchKernelEx(&cfg, dots_update2d_kernel<kYc>, A));
  } else if (A.g.dim == 3 && mode == kMarchDots && A.skel_only) {
    const bool by_point = std::getenv("ASDSM_SKEL3D_POINTS") != nullptr;
    if (by_point) {
      if (var) skel3d_dots_kernel<true><<<4 * kNumSms, 256, 0, s>>>(A);
      else skel3d_dots_kernel<false><<<4 * kNumSms, 256, 0, s>>>(A);
    } else {
      const int per_sm = std::getenv("ASDSM_DOTS3D_CTAS") ? std::atoi(std::getenv("ASDSM_DOTS3D_CTAS")) : 6;  // 6 per SM measured best (4: +7 %, 8: same)
      if (var) skel3d_dots_rows_kernel<true><<<per_sm * kNumSms, 256, 0, s>>>(A);
      else skel3d_dots_rows_kernel<false><<<per_sm * kNumSms, 256, 0, s>>>(A);
    }
  } else if (A.g.dim == 2 && mode == kMarchDots && A.skel_only) {
    if (var) skel2d_dots_kernel<true><<<kNumSms, 128, 0, s>>>(A);
    else skel2d_dots_kernel<false><<<kNumSms, 128, 0, s>>>(A);
  } else if ((mode == kMarchUpdate || mode == kMarchResidual) && ym_supported(A) && std::getenv("ASDSM_YC2D") == nullptr) {
    // the lean y-march (constant coefficients; ASDSM_YC2D=1 selects the tile-walking kernel)
    if (mode == kMarchResidual) launch_ym<kMarchResidual>(A, s);
    else launch_ym<kMarchUpdate>(A, s);
  } else if (A.g.dim == 2) {
    // measured (configs 1-2): 8-row segments, a persistent grid of 4 CTAs per SM (more CTAs
    // pay in the completion count and block scheduling, fewer leave HBM latency exposed)
    // measured (configs 1-2, one box): 4-row segments on a 4-CTA/SM persistent grid, so every
    // CTA walks ~2 tiles (config 1) and L2-prefetches the next one -- config 1 update pass 18.0 ->
    // 15.0 us, config 2 245 -> 153 us against 8-row segments (80 registers with the prefetch:
    // three CTAs per SM, a second wave at config 1); ASDSM_YC / ASDSM_YC_CPS override
    const int yc_env = std::getenv("ASDSM_YC") ? std::atoi(std::getenv("ASDSM_YC")) : 4;
    const int cps = std::getenv("ASDSM_YC_CPS") ? std::atoi(std::getenv("ASDSM_YC_CPS")) : 4;
    const int kYc = yc_env == 8 ? 8 : (yc_env == 2 ? 2 : 4);
    const long long tiles = static_cast<long long>((A.g.ext[0] + 31) / 32) * ((A.g.ext[1] + 8 * kYc - 1) / (8 * kYc));
    const unsigned nb2 = static_cast<unsigned>(std::min<long long>(tiles, static_cast<long long>(cps) * kNumSms));
#define ASDSM_YC_DISPATCH(YCV)                                                                              \
  do {                                                                                                      \
    if (var) {                                                                                              \
      if (mode == kMarchResidual) launch_pdl(stencil2d_yc_kernel<kMarchResidual, true, YCV>, nb2, 256, 0, s, A); \
      else if (mode == kMarchUpdate) launch_pdl(stencil2d_yc_kernel<kMarchUpdate, true, YCV>, nb2, 256, 0, s, A); \
      else launch_pdl(stencil2d_yc_kernel<kMarchDots, true, YCV>, nb2, 256, 0, s, A);                      \
    } else {                                                                                                \
      if (mode == kMarchResidual) launch_pdl(stencil2d_yc_kernel<kMarchResidual, false, YCV>, nb2, 256, 0, s, A); \
      else if (mode == kMarchUpdate) launch_pdl(stencil2d_yc_kernel<kMarchUpdate, false, YCV>, nb2, 256, 0, s, A); \
      else launch_pdl(stencil2d_yc_kernel<kMarchDots, false, YCV>, nb2, 256, 0, s, A);                     \
    }                                                                                                       \
  } while (0)
    if (kYc == 4) ASDSM_YC_DISPATCH(4);
    else if (kYc == 2) ASDSM_YC_DISPATCH(2);
    else ASDSM_YC_DISPATCH(8);
#undef ASDSM_YC_DISPATCH
  } else if ((mode == kMarchUpdate || mode == kMarchResidual) && stream3d_supported(A) &&
             std::getenv("ASDSM_MARCH3D") == nullptr) {
    launch_stream3d(mode, A, s);
    return;
  } else if ((mode == kMarchUpdate || mode == kMarchResidual) && zm_supported(A) && std::getenv("ASDSM_MARCH3D") == nullptr &&
             std::getenv("ASDSM_ZC3D") == nullptr) {
    // the lean z-march (constant coefficients): the residual, and the update as axpy + candidate
    // residual -- measured in the captured solve (one box, alternating): config 4 53.74 (z-coarsened
    // tile kernel) -> 50.85 (fused update, 40 B per point: 1126 us) -> 50.35 ms (two passes, 48 B);
    // config 3 11.75 -> 11.03 -> 10.9 ms.  ASDSM_UPD3D_FUSED=1 selects the fused form (read at capture).
    if (mode == kMarchResidual) {
      launch_zm<kMarchResidual>(A, s);
    } else if (std::getenv("ASDSM_UPD3D_FUSED") == nullptr) {
      axpy_update_kernel<<<8 * kNumSms, 256, 0, s>>>(A);
      ASDSM_CUDA_CHECK(cudaGetLastError());
      ++g_kernel_launches;
      launch_zm<kMarchCand>(A, s);
    } else {
      launch_zm<kMarchUpdate>(A, s);
    }
  } else if (mode == kMarchUpdate && std::getenv("ASDSM_MARCH3D") == nullptr) {
    // variable coefficients / sparse residual: axpy + candidate residual (measured against the
    // fused z-coarsened update)
    axpy_update_kernel<<<8 * kNumSms, 256, 0, s>>>(A);
    ASDSM_CUDA_CHECK(cudaGetLastError());
    ++g_kernel_launches;
    const unsigned nbz = 8 * kNumSms;
    if (var) stencil3d_zc_kernel<kMarchCand, true><<<nbz, 256, 0, s>>>(A);
    else stencil3d_zc_kernel<kMarchCand, false><<<nbz, 256, 0, s>>>(A);
  } else if (std::getenv("ASDSM_MARCH3D") == nullptr && mode != kMarchUpdate) {
    // measured (config 3/4): the barrier-free z-coarsened pass streams the residual and the
    // dot-product passes faster; the smem-plane march is faster for the 5-array update pass
    const unsigned nbz = 8 * kNumSms;
    ASDSM_MARCH_DISPATCH(stencil3d_zc_kernel, nbz, 256);
  } else {
    ASDSM_MARCH_DISPATCH(march3d_kernel, nb, TX3 * TY3);
  }
#undef ASDSM_MARCH_DISPATCH
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
