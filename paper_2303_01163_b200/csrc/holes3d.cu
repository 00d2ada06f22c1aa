// 3D error-mode hole fill.  The hole rhs 0 - A_ff*skeleton lives on the six faces of each
// hole box, so its forward transform (Wx along x, Wy along y) splits exactly into
//   x-faces  A0/A1(j,t):  Wx[k][0] (Wy A0)(l,t) + Wx[k][m0-1] (Wy A1)(l,t)
//   y-faces  B0/B1(i,t):  Wy[l][0] (Wx B0)(k,t) + Wy[l][m1-1] (Wx B1)(k,t)   (x-face points excluded)
//   z-faces  C0/C1(i,j):  [t==0] (Wx C0 Wy^T)(k,l) + [t==m2-1] (Wx C1 Wy^T)(k,l) (x/y-face points excluded)
// O(m^3) per hole instead of the dense O(m^4).  Kernel 1 (one CTA per hole) forms and
// transforms the faces; kernel 2 (one thread per (hole, k, l) line) builds the mode rhs on
// the fly and runs both Thomas sweeps along the line axis; the back transforms are DMMA GEMMs.
#include "holes3d.cuh"

namespace asdsm_b200 {

namespace {

struct HoleCtx {
  int ox, oy, oz;
};

// 0 - row_dot(p, skeleton) at hole point (i,j,t): CSR column order (fdm.cpp:110-117)
__device__ __forceinline__ double ring3(const double* __restrict__ e, const Hole3DArgs& A, const HoleCtx& h, int i,
                                        int j, int t) {
  const Stencil& st = A.st;
  const i64 sy = A.nf[0], sz = static_cast<i64>(A.nf[0]) * A.nf[1];
  const i64 p = (h.ox + i) + (h.oy + j) * sy + (h.oz + t) * sz;
  double acc = 0.0;
  if (t == 0 && h.oz > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[2], e[p - sz]));
  if (j == 0 && h.oy > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[1], e[p - sy]));
  if (i == 0 && h.ox > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[0], e[p - 1]));
  if (i == A.m[0] - 1 && h.ox + A.m[0] < A.nf[0] && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(st.right[0], e[p + 1]));
  if (j == A.m[1] - 1 && h.oy + A.m[1] < A.nf[1] && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(st.right[1], e[p + sy]));
  if (t == A.m[2] - 1 && h.oz + A.m[2] < A.nf[2] && st.has_right[2]) acc = __dadd_rn(acc, __dmul_rn(st.right[2], e[p + sz]));
  return __dsub_rn(0.0, acc);
}

__global__ void __launch_bounds__(256) hole3d_faces_kernel(const double* __restrict__ e, Hole3DArgs A,
                                                           const DevState* S) {
  if (!S->active || !S->have_e) return;
  extern __shared__ double sm[];
  const int m0 = A.m[0], m1 = A.m[1], m2 = A.m[2];
  double* sWx = sm;                // [k][i]
  double* sWy = sWx + m0 * m0;     // [l][j]
  const int mm = max(m0, max(m1, m2));
  double* F = sWy + m1 * m1;       // face staging, mm*mm
  double* G = F + mm * mm;         // temp for the z-face 2D transform, mm*mm
  for (int q = threadIdx.x; q < m0 * m0; q += blockDim.x) cp_async8(sWx + q, A.Wx + q);
  for (int q = threadIdx.x; q < m1 * m1; q += blockDim.x) cp_async8(sWy + q, A.Wy + q);
  cp_async_wait_all();
  int b = blockIdx.x;
  HoleCtx h;
  const int hx = b % A.nbox[0];
  b /= A.nbox[0];
  const int hy = b % A.nbox[1];
  const int hz = b / A.nbox[1];
  h.ox = hx * A.n[0];
  h.oy = hy * A.n[1];
  h.oz = hz * A.n[2];
  const size_t per = hole3d_face_doubles(A);
  double* out = A.faces + static_cast<i64>(blockIdx.x) * per;
  double* YA = out;                         // 2 x [t][l]
  double* XB = YA + 2 * m2 * m1;            // 2 x [t][k]
  double* CH = XB + 2 * m2 * m0;            // 2 x [l][k]
  __syncthreads();
  // x-faces: A(j,t) = f(i_face, j, t); YA[t][l] = sum_j Wy[l][j] A(j,t)
  for (int face = 0; face < (m0 > 1 ? 2 : 1); ++face) {
    const int iface = face == 0 ? 0 : m0 - 1;
    for (int q = threadIdx.x; q < m1 * m2; q += blockDim.x) {
      const int j = q % m1, t = q / m1;
      F[t * m1 + j] = ring3(e, A, h, iface, j, t);
    }
    __syncthreads();
    for (int q = threadIdx.x; q < m1 * m2; q += blockDim.x) {
      const int l = q % m1, t = q / m1;
      double acc = 0.0;
      for (int j = 0; j < m1; ++j) acc = fma(sWy[l * m1 + j], F[t * m1 + j], acc);
      YA[face * m2 * m1 + t * m1 + l] = acc;
    }
    __syncthreads();
  }
  if (m0 == 1)
    for (int q = threadIdx.x; q < m1 * m2; q += blockDim.x) YA[m2 * m1 + q] = 0.0;
  // y-faces (x-face points excluded): B(i,t) = f(i, j_face, t), 0 < i < m0-1
  for (int face = 0; face < 2; ++face) {
    const int jface = face == 0 ? 0 : m1 - 1;
    const bool active = face == 0 || m1 > 1;
    for (int q = threadIdx.x; q < m0 * m2; q += blockDim.x) {
      const int i = q % m0, t = q / m0;
      F[t * m0 + i] = (active && i > 0 && i < m0 - 1) ? ring3(e, A, h, i, jface, t) : 0.0;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < m0 * m2; q += blockDim.x) {
      const int k = q % m0, t = q / m0;
      double acc = 0.0;
      for (int i = 0; i < m0; ++i) acc = fma(sWx[k * m0 + i], F[t * m0 + i], acc);
      XB[face * m2 * m0 + t * m0 + k] = acc;
    }
    __syncthreads();
  }
  // z-faces (x/y-face points excluded): C(i,j) = f(i, j, t_face); CH[l][k] = (Wx C Wy^T)(k,l)
  for (int face = 0; face < 2; ++face) {
    const int tface = face == 0 ? 0 : m2 - 1;
    const bool active = face == 0 || m2 > 1;
    for (int q = threadIdx.x; q < m0 * m1; q += blockDim.x) {
      const int i = q % m0, j = q / m0;
      F[j * m0 + i] = (active && i > 0 && i < m0 - 1 && j > 0 && j < m1 - 1) ? ring3(e, A, h, i, j, tface) : 0.0;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < m0 * m1; q += blockDim.x) {  // G[j][k] = sum_i Wx[k][i] C(i,j)
      const int k = q % m0, j = q / m0;
      double acc = 0.0;
      for (int i = 0; i < m0; ++i) acc = fma(sWx[k * m0 + i], F[j * m0 + i], acc);
      G[j * m0 + k] = acc;
    }
    __syncthreads();
    for (int q = threadIdx.x; q < m0 * m1; q += blockDim.x) {  // CH[l][k] = sum_j Wy[l][j] G[j][k]
      const int k = q % m0, l = q / m0;
      double acc = 0.0;
      for (int j = 0; j < m1; ++j) acc = fma(sWy[l * m1 + j], G[j * m0 + k], acc);
      CH[face * m1 * m0 + l * m0 + k] = acc;
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(128) hole3d_thomas_kernel(double* __restrict__ modes, Hole3DArgs A,
                                                            const DevState* S) {
  if (!S->active || !S->have_e) return;
  const int m0 = A.m[0], m1 = A.m[1], m2 = A.m[2];
  const int ncombo = m0 * m1;
  const i64 line = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  const i64 nholes = static_cast<i64>(A.nbox[0]) * A.nbox[1] * A.nbox[2];
  if (line >= nholes * ncombo) return;
  const i64 hole = line / ncombo;
  const int combo = static_cast<int>(line % ncombo);
  const int k = combo % m0, l = combo / m0;
  const size_t per = hole3d_face_doubles(A);
  const double* __restrict__ YA = A.faces + hole * per;
  const double* __restrict__ XB = YA + 2 * m2 * m1;
  const double* __restrict__ CH = XB + 2 * m2 * m0;
  const double wx0 = __ldg(A.Wx + k * m0), wx1 = m0 > 1 ? __ldg(A.Wx + k * m0 + m0 - 1) : 0.0;
  const double wy0 = __ldg(A.Wy + l * m1), wy1 = m1 > 1 ? __ldg(A.Wy + l * m1 + m1 - 1) : 0.0;
  const double ch0 = __ldg(CH + l * m0 + k), ch1 = m2 > 1 ? __ldg(CH + m1 * m0 + l * m0 + k) : 0.0;
  const double* __restrict__ ipiv = A.ipiv;
  const double* __restrict__ cpv = A.cp;
  double* out = modes + hole * static_cast<i64>(ncombo) * m2;
  const double lft = A.line_left;
  double y = 0.0;
  for (int t = 0; t < m2; ++t) {
    double f = wx0 * __ldg(YA + t * m1 + l);
    f = fma(wx1, __ldg(YA + m2 * m1 + t * m1 + l), f);
    f = fma(wy0, __ldg(XB + t * m0 + k), f);
    f = fma(wy1, __ldg(XB + m2 * m0 + t * m0 + k), f);
    if (t == 0) f += ch0;
    if (t == m2 - 1 && m2 > 1) f += ch1;
    const double iv = __ldg(ipiv + static_cast<i64>(t) * ncombo + combo);
    y = (t == 0) ? f * iv : (f - lft * y) * iv;
    out[static_cast<i64>(t) * ncombo + combo] = y;
  }
  double x = y;
  for (int t = m2 - 2; t >= 0; --t) {
    x = out[static_cast<i64>(t) * ncombo + combo] - __ldg(cpv + static_cast<i64>(t) * ncombo + combo) * x;
    out[static_cast<i64>(t) * ncombo + combo] = x;
  }
}

}  // namespace

static size_t faces_smem(const Hole3DArgs& A) {
  const int mm = std::max(A.m[0], std::max(A.m[1], A.m[2]));
  return sizeof(double) * (static_cast<size_t>(A.m[0]) * A.m[0] + static_cast<size_t>(A.m[1]) * A.m[1] +
                           2 * static_cast<size_t>(mm) * mm);
}

void hole3d_prepare(const Hole3DArgs& A) {
  static size_t set = 48 * 1024;
  const size_t smem = faces_smem(A);
  if (smem > 220 * 1024) throw AsdsmError(kUnsupported, "3D hole faces exceed shared memory");
  if (smem > set) {
    ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole3d_faces_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem)));
    set = smem;
  }
}

void launch_hole3d_faces(const double* e, const Hole3DArgs& A, DevState* st, cudaStream_t s) {
  const size_t smem = faces_smem(A);
  const unsigned nh = static_cast<unsigned>(A.nbox[0] * A.nbox[1] * A.nbox[2]);
  hole3d_faces_kernel<<<nh, 256, smem, s>>>(e, A, st);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_hole3d_thomas(double* modes, const Hole3DArgs& A, DevState* st, cudaStream_t s) {
  const i64 lines = static_cast<i64>(A.nbox[0]) * A.nbox[1] * A.nbox[2] * A.m[0] * A.m[1];
  hole3d_thomas_kernel<<<static_cast<unsigned>((lines + 127) / 128), 128, 0, s>>>(modes, A, st);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
