// Variable-coefficient direct solves on the device: block Thomas along the box's longest
// axis with host-precomputed Schur-complement inverses (varcoef.cpp).  One CTA per box;
// thread i owns in-plane row i of every block; the dense block products read Dinv
// column-major so consecutive threads read consecutive addresses.
#include "vthomas.cuh"

namespace asdsm_b200 {

namespace {

__global__ void block_thomas_kernel(BTDev T, BoxArray A, const DevState* S) {
  if (!S->active || !S->have_e) return;
  extern __shared__ double sh[];
  double* v = sh;           // rhs / previous solution block
  const int B = T.B, nb = T.nb, L = T.L;
  const int box = blockIdx.x;
  const int bx = box % A.nbox[0], by = (box / A.nbox[0]) % A.nbox[1], bz = box / (A.nbox[0] * A.nbox[1]);
  double* base = A.ptr + bx * A.box_stride[0] + by * A.box_stride[1] + bz * A.box_stride[2];
  int oax[2] = {-1, -1}, no = 0;
  for (int a = 0; a < T.dim; ++a)
    if (a != L) oax[no++] = a;
  const int i = threadIdx.x;
  i64 off = 0;
  if (i < B) {
    const int q0 = i % T.ext[oax[0]];
    off = q0 * A.stride[oax[0]];
    if (no > 1) off += (i / T.ext[oax[0]]) * A.stride[oax[1]];
  }
  const i64 sL = A.stride[L];
  const double* Dv = T.dinv + static_cast<i64>(box) * nb * B * B;
  const double* lo = T.lo + static_cast<i64>(box) * nb * B;
  const double* up = T.up + static_cast<i64>(box) * nb * B;
  // forward: y_j = Dinv_j (b_j - l_j .* y_{j-1})
  double yprev = 0.0;
  for (int j = 0; j < nb; ++j) {
    if (i < B) {
      const double bj = base[off + j * sL];
      v[i] = j == 0 ? bj : bj - lo[static_cast<i64>(j) * B + i] * yprev;
    }
    __syncthreads();
    if (i < B) {
      const double* D = Dv + static_cast<i64>(j) * B * B;
      double acc = 0.0;
      for (int k = 0; k < B; ++k) acc = fma(D[static_cast<i64>(k) * B + i], v[k], acc);
      yprev = acc;
      base[off + j * sL] = acc;
    }
    __syncthreads();
  }
  // backward: x_j = y_j - Dinv_j (r_j .* x_{j+1})
  double xnext = yprev;
  for (int j = nb - 2; j >= 0; --j) {
    if (i < B) v[i] = up[static_cast<i64>(j) * B + i] * xnext;
    __syncthreads();
    if (i < B) {
      const double* D = Dv + static_cast<i64>(j) * B * B;
      double acc = 0.0;
      for (int k = 0; k < B; ++k) acc = fma(D[static_cast<i64>(k) * B + i], v[k], acc);
      const double x = base[off + j * sL] - acc;
      base[off + j * sL] = x;
      xnext = x;
    }
    __syncthreads();
  }
}

template <int DIM>
__global__ void hole_rhs_var_kernel(double* e, const double* b, FineGeom g, const double* coef, MeshDev m,
                                    const DevState* state) {
  if (!state->active || !state->have_e) return;
  const i64 N = g.size;
  for (i64 p = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; p < N; p += static_cast<i64>(gridDim.x) * blockDim.x) {
    const int i = static_cast<int>(p % g.ext[0]);
    const int j = static_cast<int>((p / g.ext[0]) % g.ext[1]);
    const int k = DIM == 3 ? static_cast<int>(p / (static_cast<i64>(g.ext[0]) * g.ext[1])) : 0;
    const int idx[3] = {i, j, k};
    bool hole = true;
    for (int a = 0; a < DIM; ++a)
      if ((idx[a] + 1) % m.n[a] == 0) hole = false;
    if (!hole) continue;
    // row_dot in CSR column order over skeleton neighbours (hole neighbours carry 0)
    double acc = 0.0;
    int slot = 0;
    for (int a = DIM - 1; a >= 0; --a, ++slot)
      if (idx[a] > 0 && (idx[a]) % m.n[a] == 0)  // neighbour idx-1 is on a coarse plane
        acc = __dadd_rn(acc, __dmul_rn(coef[slot * N + p], e[p - g.stride[a]]));
    ++slot;  // diag: the point itself is a hole point (0)
    for (int a = 0; a < DIM; ++a, ++slot)
      if (idx[a] < g.ext[a] - 1 && (idx[a] + 2) % m.n[a] == 0)
        acc = __dadd_rn(acc, __dmul_rn(coef[slot * N + p], e[p + g.stride[a]]));
    e[p] = __dsub_rn(b ? b[p] : 0.0, acc);
  }
}

}  // namespace

void launch_block_thomas(const BTDev& T, const BoxArray& arr, DevState* st, cudaStream_t s) {
  const unsigned nboxes = static_cast<unsigned>(arr.nbox[0] * arr.nbox[1] * arr.nbox[2]);
  const int threads = ((T.B + 31) / 32) * 32;
  block_thomas_kernel<<<nboxes, threads, sizeof(double) * T.B, s>>>(T, arr, st);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_hole_rhs_var(int dim, double* e, const double* b, const FineGeom& g, const double* coef,
                         const MeshDev& m, DevState* state, cudaStream_t s) {
  const unsigned nb = static_cast<unsigned>(std::min<i64>((g.size + 255) / 256, 8 * kNumSms));
  if (dim == 2) hole_rhs_var_kernel<2><<<nb, 256, 0, s>>>(e, b, g, coef, m, state);
  else hole_rhs_var_kernel<3><<<nb, 256, 0, s>>>(e, b, g, coef, m, state);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
