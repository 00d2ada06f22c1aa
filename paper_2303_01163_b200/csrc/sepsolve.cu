// Separable direct solver kernels for sm_100a (fp64):
//   transform_kernel : apply a dense m x m eigenvector matrix along one axis of a batch of
//                      boxes -- a register-tiled fp64 GEMM over strided lines
//   thomas_kernel    : shifted tridiagonal / bidiagonal line solves, one thread per line,
//                      precomputed pivots (coalesced across lines)
//   pcr_kernel       : parallel cyclic reduction for few long lines, one CTA per line,
//                      precomputed elimination factors, line held in shared memory
#include "sepsolve.cuh"
#include "dmma_gemm.cuh"
#include "partsolve.cuh"

#include <algorithm>
#include <cstdlib>
#include <type_traits>

namespace asdsm_b200 {

namespace {

constexpr int TP = 64, TQ = 64, TK = 16, NT = 256;
constexpr int kPcrMaxSmem = 200 * 1024;

template <typename T>
struct Acc {
  using type = T;
};

template <typename A, typename B>
struct AccOf {
  using type = cplx;
};
template <>
struct AccOf<double, double> {
  using type = double;
};

__device__ __forceinline__ void store_out(double* p, double v) { *p = v; }
__device__ __forceinline__ void store_out(double* p, cplx v) { *p = v.re; }
__device__ __forceinline__ void store_out(cplx* p, cplx v) { *p = v; }
__device__ __forceinline__ void store_out(cplx* p, double v) { *p = cplx{v, 0.0}; }

struct LineMap {
  int o_ext[2];
  i64 o_in[2], o_out[2];
  int nbox[3];
  i64 in_bs[3], out_bs[3];
  i64 nlines;
};

__device__ __forceinline__ void line_bases(const LineMap& M, i64 p, i64& ib, i64& ob) {
  const i64 o0 = p % M.o_ext[0];
  i64 t = p / M.o_ext[0];
  const i64 o1 = t % M.o_ext[1];
  t /= M.o_ext[1];
  const i64 h0 = t % M.nbox[0];
  t /= M.nbox[0];
  const i64 h1 = t % M.nbox[1];
  const i64 h2 = t / M.nbox[1];
  ib = h0 * M.in_bs[0] + h1 * M.in_bs[1] + h2 * M.in_bs[2] + o0 * M.o_in[0] + o1 * M.o_in[1];
  ob = h0 * M.out_bs[0] + h1 * M.out_bs[1] + h2 * M.out_bs[2] + o0 * M.o_out[0] + o1 * M.o_out[1];
}

// Short axes (m <= kSmallModes, e.g. the coarse axis of a slab): one thread per line, the m
// inputs in registers, the m x m matrix in shared memory -- the pass is a pure stream (the tiled
// GEMMs spend a 64-wide output tile on m outputs).  32-bit line decomposition.
constexpr int kSmallModes = 16;
__global__ void __launch_bounds__(256) small_transform_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                              const double* __restrict__ mat, int m, i64 in_es,
                                                              i64 out_es, LineMap M) {
  __shared__ double sm[kSmallModes * kSmallModes];
  for (int q = threadIdx.x; q < m * m; q += blockDim.x) sm[q] = mat[q];
  __syncthreads();
  const int n = static_cast<int>(M.nlines);
  const int e0 = M.o_ext[0], e1 = M.o_ext[1], b0 = M.nbox[0], b1 = M.nbox[1];
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < n; p += gridDim.x * blockDim.x) {
    int t = p;
    const int o0 = t % e0;
    t /= e0;
    const int o1 = t % e1;
    t /= e1;
    const int h0 = t % b0;
    t /= b0;
    const int h1 = t % b1;
    const int h2 = t / b1;
    const i64 ib = h0 * M.in_bs[0] + h1 * M.in_bs[1] + h2 * M.in_bs[2] + o0 * M.o_in[0] + o1 * M.o_in[1];
    const i64 ob = h0 * M.out_bs[0] + h1 * M.out_bs[1] + h2 * M.out_bs[2] + o0 * M.o_out[0] + o1 * M.o_out[1];
    double x[kSmallModes];
#pragma unroll
    for (int k = 0; k < kSmallModes; ++k) x[k] = k < m ? __ldg(in + ib + k * in_es) : 0.0;
#pragma unroll
    for (int q = 0; q < kSmallModes; ++q) {
      if (q >= m) break;
      double acc = 0.0;
#pragma unroll
      for (int k = 0; k < kSmallModes; ++k)
        if (k < m) acc = fma(x[k], sm[q * m + k], acc);
      out[ob + q * out_es] = acc;
    }
  }
}

// out(line, q) = sum_k in(line, k) * Mat[q][k]
template <typename TIn, typename TMat, typename TOut, bool kContig>
__global__ void __launch_bounds__(NT) transform_kernel(const TIn* __restrict__ in, TOut* __restrict__ out,
                                                       const TMat* __restrict__ mat, int m, i64 in_es,
                                                       i64 out_es, LineMap M) {
  using TA = typename AccOf<TIn, TMat>::type;
  __shared__ TIn As[TK][TP + 1];
  __shared__ TMat Bs[TK][TQ + 1];
  __shared__ i64 s_ib[TP], s_ob[TP];
  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  const i64 p0 = static_cast<i64>(blockIdx.x) * TP;
  const int q0 = blockIdx.y * TQ;
  if (tid < TP) {
    const i64 p = p0 + tid;
    i64 ib = 0, ob = 0;
    if (p < M.nlines) line_bases(M, p, ib, ob);
    s_ib[tid] = ib;
    s_ob[tid] = ob;
  }
  TA acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = zero_of<TA>();
  __syncthreads();
  for (int k0 = 0; k0 < m; k0 += TK) {
#pragma unroll
    for (int r = 0; r < (TP * TK) / NT; ++r) {
      const int e = tid + r * NT;
      int pl, kl;
      if (kContig) {
        pl = e / TK;
        kl = e % TK;
      } else {
        pl = e % TP;
        kl = e / TP;
      }
      const int k = k0 + kl;
      TIn v = zero_of<TIn>();
      if (p0 + pl < M.nlines && k < m) v = in[s_ib[pl] + static_cast<i64>(k) * in_es];
      As[kl][pl] = v;
    }
#pragma unroll
    for (int r = 0; r < (TQ * TK) / NT; ++r) {
      const int e = tid + r * NT;
      const int ql = e / TK, kl = e % TK;
      const int q = q0 + ql, k = k0 + kl;
      TMat v = zero_of<TMat>();
      if (q < m && k < m) v = mat[static_cast<i64>(q) * m + k];
      Bs[kl][ql] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      TIn a[4];
      TMat b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = kContig ? As[kk][ty + 16 * i] : As[kk][tx + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = kContig ? Bs[kk][tx + 16 * j] : Bs[kk][ty + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) fma_acc(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int pl = kContig ? ty + 16 * i : tx + 16 * i;
    if (p0 + pl >= M.nlines) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = q0 + (kContig ? tx + 16 * j : ty + 16 * j);
      if (q < m) store_out(&out[s_ob[pl] + static_cast<i64>(q) * out_es], acc[i][j]);
    }
  }
}

template <typename T>
struct LineArgs {
  T* data;
  i64 stride_L;
  int m;
  int ncombo;
  int cext0;
  i64 cstride0, cstride1;
  int nbox[3];
  i64 box_stride[3];
  i64 nlines;
  const T* ipiv;
  const T* cp;
  double left;
};

template <typename T>
__device__ __forceinline__ T scale_sub(T g, double l, T y) {  // g - l*y
  return g - l * y;
}
template <>
__device__ __forceinline__ double scale_sub<double>(double g, double l, double y) {
  return g - l * y;
}

template <typename T>
__global__ void thomas_kernel(LineArgs<T> A) {
  const i64 line = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (line >= A.nlines) return;
  const int combo = static_cast<int>(line % A.ncombo);
  i64 t = line / A.ncombo;
  const i64 h0 = t % A.nbox[0];
  t /= A.nbox[0];
  const i64 h1 = t % A.nbox[1];
  const i64 h2 = t / A.nbox[1];
  const int c0 = combo % A.cext0, c1 = combo / A.cext0;
  T* d = A.data + h0 * A.box_stride[0] + h1 * A.box_stride[1] + h2 * A.box_stride[2] + c0 * A.cstride0 +
         c1 * A.cstride1;
  T y = d[0] * A.ipiv[combo];
  d[0] = y;
  for (int p = 1; p < A.m; ++p) {
    const T g = d[static_cast<i64>(p) * A.stride_L];
    y = scale_sub(g, A.left, y) * A.ipiv[static_cast<i64>(p) * A.ncombo + combo];
    d[static_cast<i64>(p) * A.stride_L] = y;
  }
  T x = y;
  for (int p = A.m - 2; p >= 0; --p) {
    const T yp = d[static_cast<i64>(p) * A.stride_L];
    x = yp - A.cp[static_cast<i64>(p) * A.ncombo + combo] * x;
    d[static_cast<i64>(p) * A.stride_L] = x;
  }
}

template <typename T>
struct PcrArgs {
  T* data;
  i64 stride_L;
  int m, levels, ncombo, cext0;
  i64 cstride0, cstride1;
  int nbox[3];
  i64 box_stride[3];
  const T* k1;
  const T* k2;
  const T* invb;
};

template <typename T>
__global__ void pcr_kernel(PcrArgs<T> A) {
  extern __shared__ unsigned char smem_raw[];
  T* x0 = reinterpret_cast<T*>(smem_raw);
  T* x1 = x0 + A.m;
  const i64 line = blockIdx.x;
  const int combo = static_cast<int>(line % A.ncombo);
  i64 t = line / A.ncombo;
  const i64 h0 = t % A.nbox[0];
  t /= A.nbox[0];
  const i64 h1 = t % A.nbox[1];
  const i64 h2 = t / A.nbox[1];
  const int c0 = combo % A.cext0, c1 = combo / A.cext0;
  T* d = A.data + h0 * A.box_stride[0] + h1 * A.box_stride[1] + h2 * A.box_stride[2] + c0 * A.cstride0 +
         c1 * A.cstride1;
  for (int i = threadIdx.x; i < A.m; i += blockDim.x) x0[i] = d[static_cast<i64>(i) * A.stride_L];
  __syncthreads();
  const T* K1 = A.k1 + static_cast<i64>(combo) * A.levels * A.m;
  const T* K2 = A.k2 + static_cast<i64>(combo) * A.levels * A.m;
  int s = 1;
  for (int lev = 0; lev < A.levels; ++lev, s <<= 1) {
    for (int i = threadIdx.x; i < A.m; i += blockDim.x) {
      T v = x0[i];
      if (i - s >= 0) v = v - K1[static_cast<i64>(lev) * A.m + i] * x0[i - s];
      if (i + s < A.m) v = v - K2[static_cast<i64>(lev) * A.m + i] * x0[i + s];
      x1[i] = v;
    }
    __syncthreads();
    T* tmp = x0;
    x0 = x1;
    x1 = tmp;
  }
  const T* IB = A.invb + static_cast<i64>(combo) * A.m;
  for (int i = threadIdx.x; i < A.m; i += blockDim.x) d[static_cast<i64>(i) * A.stride_L] = x0[i] * IB[i];
}

// Lines solved by one warp each with the partition method (SepSolver::part): 8 lines per CTA,
// the lines and their tables staged in shared memory (consecutive lines are neighbours along the
// fastest combo axis, so the staging reads 8 adjacent values per line position).
constexpr int kPartWarps = 8;
struct PartArgs {
  double* data;
  i64 stride_L;
  int m, ncombo, cext0;
  i64 cstride0, cstride1;
  int nbox[3];
  i64 box_stride[3];
  i64 nlines;
  const double* part;
  int pstride, P, last;
  double l, r;
  int line_major;  // stride_L == 1: stage along the line
};

template <int SEG>
__global__ void __launch_bounds__(32 * kPartWarps) part_line_kernel(PartArgs A) {
  extern __shared__ __align__(16) double psm[];
  double* lines = psm;                        // [kPartWarps][m]
  double* tabs = psm + kPartWarps * A.m;      // [kPartWarps][pstride] (ASDSM_PART_LINE_STAGE)
  (void)tabs;
  const int warp = threadIdx.x >> 5;
  const i64 line0 = static_cast<i64>(blockIdx.x) * kPartWarps;
  auto base_of = [&](i64 line) -> double* {
    const int combo = static_cast<int>(line % A.ncombo);
    i64 t = line / A.ncombo;
    const i64 h0 = t % A.nbox[0];
    t /= A.nbox[0];
    const i64 h1 = t % A.nbox[1];
    const i64 h2 = t / A.nbox[1];
    const int c0 = combo % A.cext0, c1 = combo / A.cext0;
    return A.data + h0 * A.box_stride[0] + h1 * A.box_stride[1] + h2 * A.box_stride[2] + c0 * A.cstride0 +
           c1 * A.cstride1;
  };
  __shared__ double* bases[kPartWarps];
  if (threadIdx.x < kPartWarps) {
    const i64 line = line0 + threadIdx.x;
    bases[threadIdx.x] = line < A.nlines ? base_of(line) : nullptr;
  }
#ifdef ASDSM_PART_LINE_STAGE
  for (int q = threadIdx.x; q < kPartWarps * A.pstride; q += blockDim.x) {
    const int w = q / A.pstride, o = q - w * A.pstride;
    const i64 line = line0 + w;
    if (line < A.nlines) cp_async8(tabs + q, A.part + static_cast<i64>(line % A.ncombo) * A.pstride + o);
  }
#endif
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  __syncthreads();
  const int n = kPartWarps * A.m;
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    int w, p;
    if (A.line_major) {
      w = q / A.m;
      p = q - w * A.m;
    } else {
      p = q / kPartWarps;
      w = q - p * kPartWarps;
    }
    const double* b = bases[w];
    lines[w * A.m + p] = b ? b[static_cast<i64>(p) * A.stride_L] : 0.0;
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
#ifdef ASDSM_PART_LINE_STAGE
  if (bases[warp]) part_solve_line<SEG>(lines + warp * A.m, tabs + warp * A.pstride, A.m, A.P, A.last, A.l, A.r);
#else
  // the mode's partition table straight from L2 (measured, configs 3/4: 11.87 -> 11.79 ms,
  // 53.89 -> 53.83 ms against staging it per CTA)
  if (bases[warp])
    part_solve_line<SEG>(lines + warp * A.m, A.part + static_cast<i64>((line0 + warp) % A.ncombo) * A.pstride, A.m, A.P,
                         A.last, A.l, A.r);
#endif
  __syncthreads();
  for (int q = threadIdx.x; q < n; q += blockDim.x) {
    int w, p;
    if (A.line_major) {
      w = q / A.m;
      p = q - w * A.m;
    } else {
      p = q / kPartWarps;
      w = q - p * kPartWarps;
    }
    double* b = bases[w];
    if (b) b[static_cast<i64>(p) * A.stride_L] = lines[w * A.m + p];
  }
}

// Compact mode layout of a batch: element strides (1, e0, e0*e1), boxes back to back.
BoxArray compact_layout(const SepSolver& S, const BoxArray& like, void* ptr) {
  BoxArray b;
  b.ptr = static_cast<double*>(ptr);
  b.stride[0] = 1;
  b.stride[1] = S.ext[0];
  b.stride[2] = static_cast<i64>(S.ext[0]) * S.ext[1];
  const i64 bs = S.mode_size();
  for (int a = 0; a < 3; ++a) b.nbox[a] = like.nbox[a];
  b.box_stride[0] = bs;
  b.box_stride[1] = bs * like.nbox[0];
  b.box_stride[2] = bs * like.nbox[0] * like.nbox[1];
  return b;
}

// eo: 1 back transform (mat = V), 2 forward (mat = W): long axes with a half sine table run the
// even/odd-split DMMA kernel (half the MMAs); 0 or short axes the dense one
template <typename TIn, typename TMat, typename TOut>
void launch_transform(const SepSolver& S, int axis, const BoxArray& in, const BoxArray& out, const TMat* mat,
                      cudaStream_t st, int eo = 0) {
  LineMap M{};
  int no = 0;
  for (int a = 0; a < 3; ++a) {
    if (a == axis) continue;
    M.o_ext[no] = a < S.dim ? S.ext[a] : 1;
    M.o_in[no] = in.stride[a];
    M.o_out[no] = out.stride[a];
    ++no;
  }
  i64 nb = 1;
  for (int a = 0; a < 3; ++a) {
    M.nbox[a] = in.nbox[a];
    M.in_bs[a] = in.box_stride[a];
    M.out_bs[a] = out.box_stride[a];
    nb *= in.nbox[a];
  }
  M.nlines = static_cast<i64>(M.o_ext[0]) * M.o_ext[1] * nb;
  const int m = S.ext[axis];
  dim3 grid(static_cast<unsigned>((M.nlines + TP - 1) / TP), static_cast<unsigned>((m + TQ - 1) / TQ));
  const TIn* ip = reinterpret_cast<const TIn*>(in.ptr);
  TOut* op = reinterpret_cast<TOut*>(out.ptr);
  if constexpr (std::is_same<TIn, double>::value && std::is_same<TMat, double>::value &&
                std::is_same<TOut, double>::value) {
    const bool scalar = std::getenv("ASDSM_SCALAR_GEMM") != nullptr;
    if (m <= kSmallModes && M.nlines < (1LL << 31) && std::getenv("ASDSM_NO_SMALL_TRANSFORM") == nullptr) {
      const i64 nb = std::min<i64>((M.nlines + 255) / 256, 16LL * kNumSms);
      small_transform_kernel<<<static_cast<unsigned>(nb), 256, 0, st>>>(ip, op, mat, m, in.stride[axis], out.stride[axis], M);
      ASDSM_CUDA_CHECK(cudaGetLastError());
      ++g_kernel_launches;
      return;
    }
    if (!scalar) {
      GemmLines G{};
      for (int i = 0; i < 2; ++i) {
        G.o_ext[i] = M.o_ext[i];
        G.o_in[i] = M.o_in[i];
        G.o_out[i] = M.o_out[i];
      }
      for (int a = 0; a < 3; ++a) {
        G.nbox[a] = M.nbox[a];
        G.in_bs[a] = M.in_bs[a];
        G.out_bs[a] = M.out_bs[a];
      }
      G.nlines = M.nlines;
      const bool dense = std::getenv("ASDSM_DENSE_GEMM") != nullptr;  // (read at capture time)
      if (eo != 0 && S.half[axis] != nullptr && m >= eo_min_modes() && !dense) {
        launch_dmma_eo_transform(eo == 1, ip, op, S.half[axis], m, in.stride[axis], out.stride[axis], G, st);
        return;
      }
      launch_dmma_transform(ip, op, mat, m, in.stride[axis], out.stride[axis], G, st);
      return;
    }
  }
  if (axis == 0)
    transform_kernel<TIn, TMat, TOut, true><<<grid, NT, 0, st>>>(ip, op, mat, m, in.stride[axis], out.stride[axis], M);
  else
    transform_kernel<TIn, TMat, TOut, false><<<grid, NT, 0, st>>>(ip, op, mat, m, in.stride[axis], out.stride[axis], M);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

template <typename T>
void launch_line_solve(const SepSolver& S, const BoxArray& buf, cudaStream_t st) {
  int cax[2] = {-1, -1}, nco = 0;
  for (int a = 0; a < S.dim; ++a)
    if (a != S.L) cax[nco++] = a;
  i64 nb = static_cast<i64>(buf.nbox[0]) * buf.nbox[1] * buf.nbox[2];
  if (!S.use_pcr) {
    LineArgs<T> A{};
    A.data = reinterpret_cast<T*>(buf.ptr);
    A.stride_L = buf.stride[S.L];
    A.m = S.ext[S.L];
    A.ncombo = S.ncombo;
    A.cext0 = cax[0] >= 0 ? S.ext[cax[0]] : 1;
    A.cstride0 = cax[0] >= 0 ? buf.stride[cax[0]] : 0;
    A.cstride1 = cax[1] >= 0 ? buf.stride[cax[1]] : 0;
    for (int a = 0; a < 3; ++a) {
      A.nbox[a] = buf.nbox[a];
      A.box_stride[a] = buf.box_stride[a];
    }
    A.nlines = nb * S.ncombo;
    A.ipiv = reinterpret_cast<const T*>(S.th_ipiv);
    A.cp = reinterpret_cast<const T*>(S.th_cp);
    A.left = S.line_left;
    const int bs = 128;
    thomas_kernel<T><<<static_cast<unsigned>((A.nlines + bs - 1) / bs), bs, 0, st>>>(A);
  } else if (std::is_same<T, double>::value && S.part != nullptr && !S.complex_modes &&
             std::getenv("ASDSM_PCR_LINES") == nullptr) {  // (read at capture time)
    PartArgs A{};
    A.data = reinterpret_cast<double*>(buf.ptr);
    A.stride_L = buf.stride[S.L];
    A.m = S.ext[S.L];
    A.ncombo = S.ncombo;
    A.cext0 = cax[0] >= 0 ? S.ext[cax[0]] : 1;
    A.cstride0 = cax[0] >= 0 ? buf.stride[cax[0]] : 0;
    A.cstride1 = cax[1] >= 0 ? buf.stride[cax[1]] : 0;
    for (int a = 0; a < 3; ++a) {
      A.nbox[a] = buf.nbox[a];
      A.box_stride[a] = buf.box_stride[a];
    }
    A.nlines = nb * S.ncombo;
    A.part = S.part;
    A.pstride = S.part_stride;
    A.P = S.part_P;
    A.last = S.part_last;
    A.l = S.line_left;
    A.r = S.line_right;
    A.line_major = A.stride_L == 1 ? 1 : 0;
#ifdef ASDSM_PART_LINE_STAGE
    const size_t smem = sizeof(double) * kPartWarps * (static_cast<size_t>(A.m) + A.pstride);
#else
    const size_t smem = sizeof(double) * kPartWarps * static_cast<size_t>(A.m);
#endif
    if (smem > kPcrMaxSmem) throw AsdsmError(kUnsupported, "partitioned line solve exceeds shared memory");
    const unsigned grid = static_cast<unsigned>((A.nlines + kPartWarps - 1) / kPartWarps);
    switch (S.part_seg) {
      case 2: part_line_kernel<2><<<grid, 32 * kPartWarps, smem, st>>>(A); break;
      case 4: part_line_kernel<4><<<grid, 32 * kPartWarps, smem, st>>>(A); break;
      case 8: part_line_kernel<8><<<grid, 32 * kPartWarps, smem, st>>>(A); break;
      case 12: part_line_kernel<12><<<grid, 32 * kPartWarps, smem, st>>>(A); break;
      case 16: part_line_kernel<16><<<grid, 32 * kPartWarps, smem, st>>>(A); break;
      case 20: part_line_kernel<20><<<grid, 32 * kPartWarps, smem, st>>>(A); break;
      case 24: part_line_kernel<24><<<grid, 32 * kPartWarps, smem, st>>>(A); break;
      case 28: part_line_kernel<28><<<grid, 32 * kPartWarps, smem, st>>>(A); break;
      default: part_line_kernel<32><<<grid, 32 * kPartWarps, smem, st>>>(A); break;
    }
  } else {
    PcrArgs<T> A{};
    A.data = reinterpret_cast<T*>(buf.ptr);
    A.stride_L = buf.stride[S.L];
    A.m = S.ext[S.L];
    A.levels = S.pcr_levels;
    A.ncombo = S.ncombo;
    A.cext0 = cax[0] >= 0 ? S.ext[cax[0]] : 1;
    A.cstride0 = cax[0] >= 0 ? buf.stride[cax[0]] : 0;
    A.cstride1 = cax[1] >= 0 ? buf.stride[cax[1]] : 0;
    for (int a = 0; a < 3; ++a) {
      A.nbox[a] = buf.nbox[a];
      A.box_stride[a] = buf.box_stride[a];
    }
    A.k1 = reinterpret_cast<const T*>(S.pcr_k1);
    A.k2 = reinterpret_cast<const T*>(S.pcr_k2);
    A.invb = reinterpret_cast<const T*>(S.pcr_invb);
    const size_t smem = 2 * static_cast<size_t>(A.m) * sizeof(T);
    if (smem > kPcrMaxSmem) throw AsdsmError(kUnsupported, "PCR line longer than shared memory allows");
    pcr_kernel<T><<<static_cast<unsigned>(nb * S.ncombo), 1024, smem, st>>>(A);
  }
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace

void sep_back_transform(const SepSolver& S, void* modes, const BoxArray& out, void* scratch, cudaStream_t st) {
  if (S.complex_modes) throw AsdsmError(kUnsupported, "sep_back_transform: complex modes");
  const BoxArray c0 = compact_layout(S, out, modes);
  if (S.nd == 1) {
    launch_transform<double, double, double>(S, S.dax[0], c0, out, S.V[S.dax[0]], st, 1);
    return;
  }
  const BoxArray c1 = compact_layout(S, out, scratch);
  launch_transform<double, double, double>(S, S.dax[1], c0, c1, S.V[S.dax[1]], st, 1);
  launch_transform<double, double, double>(S, S.dax[0], c1, out, S.V[S.dax[0]], st, 1);
}

void sep_prepare() {
  static bool done = false;
  if (done) return;
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(pcr_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(pcr_kernel<cplx>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(part_line_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(part_line_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(part_line_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(part_line_kernel<12>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(part_line_kernel<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(part_line_kernel<20>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(part_line_kernel<24>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(part_line_kernel<28>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(part_line_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPcrMaxSmem));
  done = true;
}

size_t sep_scratch_bytes(const SepSolver& S, i64 nboxes) {
  return static_cast<size_t>(S.mode_size()) * nboxes * (S.complex_modes ? sizeof(cplx) : sizeof(double));
}

void sep_solve(const SepSolver& S, const BoxArray& in, const BoxArray& out, void* scratch0, void* scratch1,
               cudaStream_t st) {
  const BoxArray c0 = compact_layout(S, in, scratch0);
  const BoxArray c1 = compact_layout(S, in, scratch1);
  if (S.complex_modes) {
    // One diagonalized axis (enforced at build time).
    const int a = S.dax[0];
    launch_transform<double, cplx, cplx>(S, a, in, c0, reinterpret_cast<const cplx*>(S.W[a]), st);
    launch_line_solve<cplx>(S, c0, st);
    launch_transform<cplx, cplx, double>(S, a, c0, out, reinterpret_cast<const cplx*>(S.V[a]), st);
    return;
  }
  if (S.nd == 1) {
    const int a = S.dax[0];
    launch_transform<double, double, double>(S, a, in, c0, S.W[a], st, 2);
    launch_line_solve<double>(S, c0, st);
    launch_transform<double, double, double>(S, a, c0, out, S.V[a], st, 1);
    return;
  }
  const int a0 = S.dax[0], a1 = S.dax[1];
  launch_transform<double, double, double>(S, a0, in, c0, S.W[a0], st, 2);
  launch_transform<double, double, double>(S, a1, c0, c1, S.W[a1], st, 2);
  launch_line_solve<double>(S, c1, st);
  launch_transform<double, double, double>(S, a1, c1, c0, S.V[a1], st, 1);
  launch_transform<double, double, double>(S, a0, c0, out, S.V[a0], st, 1);
}

}  // namespace asdsm_b200
