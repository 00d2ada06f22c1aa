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

namespace asdsm_b200 {

namespace {

constexpr int TX2 = 128, SY2 = 32;            // 2D: threads per x-tile, rows per strip
constexpr int TX3 = 32, TY3 = 16, SZ3 = 16;   // 3D: x-by-y tile, z chunk

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

template <int MODE>
__global__ void __launch_bounds__(TX2) march2d_kernel(MarchArgs A) {
  DevState* S = A.state;
  if (!S->active) return;
  const int cur = S->cur;
  double s = 0.0;
  bool work = true;
  if (MODE == kMarchUpdate) {
    s = S->s;
    work = s != 0.0;
  }
  if (MODE == kMarchDots) work = S->have_e != 0;
  const int Nx = A.g.ext[0], Ny = A.g.ext[1];
  const i64 sy = A.g.stride[1];
  const Stencil& st = A.st;
  Src<MODE> V{cur ? A.u1 : A.u0, A.e, s};
  const double* __restrict__ rcur = cur ? A.r1 : A.r0;
  double* __restrict__ uo = MODE == kMarchUpdate ? (cur ? A.uo0 : A.uo1) : nullptr;
  double* __restrict__ ro = MODE == kMarchUpdate ? (cur ? A.ro0 : A.ro1) : (cur ? A.ro1 : A.ro0);
  __shared__ double row[2][TX2 + 2];
  const int ntx = (Nx + TX2 - 1) / TX2;
  const int tx = blockIdx.x % ntx, ty = blockIdx.x / ntx;
  const int x0 = tx * TX2, y0 = ty * SY2;
  const int y1 = min(y0 + SY2, Ny);
  const int t = threadIdx.x;
  const int x = x0 + t;
  const bool in = x < Nx;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;  // ssq/num, max, esq/den, emax
  if (work) {
    double vd = (in && y0 > 0) ? V(x + (y0 - 1) * sy) : 0.0;
    double vc = in ? V(x + y0 * sy) : 0.0;
    int buf = 0;
    for (int y = y0; y < y1; ++y) {
      const i64 p = x + y * sy;
      const double vu = (in && y + 1 < Ny) ? V(p + sy) : 0.0;
      row[buf][t + 1] = vc;
      if (t == 0) row[buf][0] = x0 > 0 ? V(x0 - 1 + y * sy) : 0.0;
      if (t == TX2 - 1 || x == Nx - 1) row[buf][t + 2] = x + 1 < Nx ? V(p + 1) : 0.0;
      __syncthreads();
      if (in) {
        double acc = 0.0;
        if (y > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[1], vd));
        if (x > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[0], row[buf][t]));
        acc = __dadd_rn(acc, __dmul_rn(st.diag, vc));
        if (x < Nx - 1 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(st.right[0], row[buf][t + 2]));
        if (y < Ny - 1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(st.right[1], vu));
        if (MODE == kMarchDots) {
          const double rp = __ldg(rcur + p);
          a0 += rp * acc;
          a2 += acc * acc;
        } else {
          const double r = __dsub_rn(__ldg(A.b + p), acc);
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
      vd = vc;
      vc = vu;
      buf ^= 1;
    }
  }
  block_reduce4_march(a0, a1, a2, a3, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}

template <int MODE>
__global__ void __launch_bounds__(TX3 * TY3) march3d_kernel(MarchArgs A) {
  DevState* S = A.state;
  if (!S->active) return;
  const int cur = S->cur;
  double s = 0.0;
  bool work = true;
  if (MODE == kMarchUpdate) {
    s = S->s;
    work = s != 0.0;
  }
  if (MODE == kMarchDots) work = S->have_e != 0;
  const int Nx = A.g.ext[0], Ny = A.g.ext[1], Nz = A.g.ext[2];
  const i64 sy = A.g.stride[1], sz = A.g.stride[2];
  const Stencil& st = A.st;
  Src<MODE> V{cur ? A.u1 : A.u0, A.e, s};
  const double* __restrict__ rcur = cur ? A.r1 : A.r0;
  double* __restrict__ uo = MODE == kMarchUpdate ? (cur ? A.uo0 : A.uo1) : nullptr;
  double* __restrict__ ro = MODE == kMarchUpdate ? (cur ? A.ro0 : A.ro1) : (cur ? A.ro1 : A.ro0);
  __shared__ double pl[2][TY3 + 2][TX3 + 2];
  const int ntx = (Nx + TX3 - 1) / TX3, nty = (Ny + TY3 - 1) / TY3;
  int b = blockIdx.x;
  const int bx = b % ntx;
  b /= ntx;
  const int by = b % nty;
  const int bz = b / nty;
  const int x0 = bx * TX3, y0 = by * TY3, z0 = bz * SZ3;
  const int z1 = min(z0 + SZ3, Nz);
  const int tx = threadIdx.x % TX3, ty = threadIdx.x / TX3;
  const int x = x0 + tx, y = y0 + ty;
  const bool in = x < Nx && y < Ny;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (work) {
    const i64 pxy = x + y * sy;
    double vd = (in && z0 > 0) ? V(pxy + (z0 - 1) * sz) : 0.0;
    double vc = in ? V(pxy + z0 * sz) : 0.0;
    int buf = 0;
    for (int z = z0; z < z1; ++z) {
      const i64 p = pxy + z * sz;
      const double vu = (in && z + 1 < Nz) ? V(p + sz) : 0.0;
      pl[buf][ty + 1][tx + 1] = vc;
      if (in) {
        if (tx == 0) pl[buf][ty + 1][0] = x > 0 ? V(p - 1) : 0.0;
        if (tx == TX3 - 1 || x == Nx - 1) pl[buf][ty + 1][tx + 2] = x + 1 < Nx ? V(p + 1) : 0.0;
        if (ty == 0) pl[buf][0][tx + 1] = y > 0 ? V(p - sy) : 0.0;
        if (ty == TY3 - 1 || y == Ny - 1) pl[buf][ty + 2][tx + 1] = y + 1 < Ny ? V(p + sy) : 0.0;
      }
      __syncthreads();
      if (in) {
        double acc = 0.0;
        if (z > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[2], vd));
        if (y > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[1], pl[buf][ty][tx + 1]));
        if (x > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[0], pl[buf][ty + 1][tx]));
        acc = __dadd_rn(acc, __dmul_rn(st.diag, vc));
        if (x < Nx - 1 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(st.right[0], pl[buf][ty + 1][tx + 2]));
        if (y < Ny - 1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(st.right[1], pl[buf][ty + 2][tx + 1]));
        if (z < Nz - 1 && st.has_right[2]) acc = __dadd_rn(acc, __dmul_rn(st.right[2], vu));
        if (MODE == kMarchDots) {
          const double rp = __ldg(rcur + p);
          a0 += rp * acc;
          a2 += acc * acc;
        } else {
          const double r = __dsub_rn(__ldg(A.b + p), acc);
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
      vd = vc;
      vc = vu;
      buf ^= 1;
    }
  }
  block_reduce4_march(a0, a1, a2, a3, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}

}  // namespace

unsigned march_blocks(const FineGeom& g) {
  if (g.dim == 2) return static_cast<unsigned>(((g.ext[0] + TX2 - 1) / TX2) * ((g.ext[1] + SY2 - 1) / SY2));
  return static_cast<unsigned>(((g.ext[0] + TX3 - 1) / TX3) * ((g.ext[1] + TY3 - 1) / TY3) * ((g.ext[2] + SZ3 - 1) / SZ3));
}

void launch_march(int mode, const MarchArgs& A, cudaStream_t s) {
  const unsigned nb = march_blocks(A.g);
  if (nb > static_cast<unsigned>(kRedStride)) throw AsdsmError(kUnsupported, "fine grid too large for the partial buffer");
  if (A.g.dim == 2) {
    if (mode == kMarchResidual) march2d_kernel<kMarchResidual><<<nb, TX2, 0, s>>>(A);
    else if (mode == kMarchUpdate) march2d_kernel<kMarchUpdate><<<nb, TX2, 0, s>>>(A);
    else march2d_kernel<kMarchDots><<<nb, TX2, 0, s>>>(A);
  } else {
    if (mode == kMarchResidual) march3d_kernel<kMarchResidual><<<nb, TX3 * TY3, 0, s>>>(A);
    else if (mode == kMarchUpdate) march3d_kernel<kMarchUpdate><<<nb, TX3 * TY3, 0, s>>>(A);
    else march3d_kernel<kMarchDots><<<nb, TX3 * TY3, 0, s>>>(A);
  }
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
