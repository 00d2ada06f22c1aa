// 2D slab solves (the anisotropic systems A_fc, A_cf of Alg. 1, solved by the reference with
// Eigen SparseLU, linsolve.cpp:58-66) as the paper's dimension-reduced line solves:
//   launch 1, one CTA per (coarse mode k, slab): restriction of r onto the slab fused with the
//            coarse-axis eigenvector transform, then PCR along the fine line in shared memory;
//   launch 2: back transform to the slab layout + squared norms for normalize_or_throw
//            (solver.cpp:79-84), the last block finalizing both norms.
#include "slab2d.cuh"
#include "ctrl.cuh"
#include "skel2d.cuh"

#include <type_traits>

namespace asdsm_b200 {

namespace {

constexpr int kThreads = 1024;
constexpr int kMaxSmem = 220 * 1024;
constexpr int kSlabWBytes = 24 * 16;                 // station weights (nc <= 24, complex)
constexpr int kSlabWOffset = kMaxSmem - kSlabWBytes;  // at the top of the dynamic area

template <typename T>
__device__ __forceinline__ T ld(const double* p, i64 i);
template <>
__device__ __forceinline__ double ld<double>(const double* p, i64 i) { return __ldg(p + i); }
template <>
__device__ __forceinline__ cplx ld<cplx>(const double* p, i64 i) { return cplx{__ldg(p + 2 * i), __ldg(p + 2 * i + 1)}; }

__device__ __forceinline__ void st_out(double* p, i64 i, double v) { p[i] = v; }
__device__ __forceinline__ void st_out(double* p, i64 i, cplx v) { reinterpret_cast<cplx*>(p)[i] = v; }

#ifdef ASDSM_SLAB_TRACE
#define SLAB_STAMP(i) T_[i] = clock64()
#define SLAB_TRACE_DECL long long T_[6] = {clock64(), 0, 0, 0, 0, 0};
#else
#define SLAB_STAMP(i)
#define SLAB_TRACE_DECL
#endif

template <typename T>
__global__ void __launch_bounds__(kThreads) slab2d_fwd_kernel(Slab2DArgs A, const DevState* S) {
  if (!S->active) return;
  SLAB_TRACE_DECL
  extern __shared__ unsigned char smem[];
  const int a = blockIdx.y, f = 1 - a;
  const MeshDev& m = A.m;
  const int nc = m.nc[a], nf = m.nf[f], k = blockIdx.x;
  if (k >= nc) return;
  T* x0 = reinterpret_cast<T*>(smem);
  T* x1 = x0 + nf;
  const int L = A.levels[a];
  const double* K1 = A.k1[a];
  const double* K2 = A.k2[a];
  if (std::is_same<T, double>::value && A.pcr_smem) {
    // every level's factors bulk-loaded next to the line, in flight during the gather
    double* sk1 = reinterpret_cast<double*>(x1 + nf);
    double* sk2 = sk1 + static_cast<i64>(L) * nf;
    const i64 base = static_cast<i64>(k) * L * nf;
    for (int i = threadIdx.x; i < L * nf; i += blockDim.x) {
      cp_async8(sk1 + i, K1 + base + i);
      cp_async8(sk2 + i, K2 + base + i);
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  }
  const double* rf = A.in_fine0 ? (S->cur ? A.in_fine1 : A.in_fine0) : nullptr;
  const double* rs = A.sta0 ? (S->cur ? A.sta1 : A.sta0) + (a == 0 ? 0 : static_cast<i64>(m.nc[0]) * m.nf[1]) : nullptr;
  const i64 Nx = m.nf[0];
  // station weights W[k][:] staged in shared memory (broadcast reads), after the PCR area
  T* sw = reinterpret_cast<T*>(smem + kSlabWOffset);
  for (int j = threadIdx.x; j < nc; j += blockDim.x) sw[j] = ld<T>(A.W[a], static_cast<i64>(k) * nc + j);
  __syncthreads();
  constexpr int kChunk = 10;  // station values of one fine point in flight at once
  for (int x = threadIdx.x; x < nf; x += blockDim.x) {
    T acc = zero_of<T>();
    for (int j0 = 0; j0 < nc; j0 += kChunk) {
      double v[kChunk];
#pragma unroll
      for (int q = 0; q < kChunk; ++q) {
        const int j = j0 + q;
        v[q] = 0.0;
        if (j < nc) {
          if (rs) v[q] = __ldg(rs + static_cast<i64>(j) * nf + x);
          else if (rf) {
            const int fj = (j + 1) * m.n[a] - 1;  // station on the coarse axis
            v[q] = (a == 0) ? __ldg(rf + fj + Nx * x) : __ldg(rf + x + Nx * fj);
          } else {
            v[q] = (a == 0) ? __ldg(A.in_slab[a] + j + static_cast<i64>(nc) * x) : __ldg(A.in_slab[a] + x + static_cast<i64>(nf) * j);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < kChunk; ++q)
        if (j0 + q < nc) fma_acc(acc, sw[j0 + q], v[q]);
    }
    x0[x] = acc;
  }
  __syncthreads();
  SLAB_STAMP(1);
  if constexpr (std::is_same<T, cplx>::value) {  // complex: coefficients straight from L2
    int s = 1;
    for (int lev = 0; lev < L; ++lev, s <<= 1) {
      const i64 base = (static_cast<i64>(k) * L + lev) * nf;
      for (int i = threadIdx.x; i < nf; i += blockDim.x) {
        T v = x0[i];
        if (i - s >= 0) v = v - ld<T>(K1, base + i) * x0[i - s];
        if (i + s < nf) v = v - ld<T>(K2, base + i) * x0[i + s];
        x1[i] = v;
      }
      __syncthreads();
      T* t = x0;
      x0 = x1;
      x1 = t;
    }
    for (int i = threadIdx.x; i < nf; i += blockDim.x)
      st_out(A.modes[a], static_cast<i64>(k) * nf + i, x0[i] * ld<T>(A.invb[a], static_cast<i64>(k) * nf + i));
    return;
  }
  if (A.pcr_smem) {  // pure shared-memory PCR over the staged factors
    double* sk1 = reinterpret_cast<double*>(x1 + nf);
    double* sk2 = sk1 + static_cast<i64>(L) * nf;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    SLAB_STAMP(2);
    int s = 1;
    for (int lev = 0; lev < L; ++lev, s <<= 1) {
      const double* c1 = sk1 + static_cast<i64>(lev) * nf;
      const double* c2 = sk2 + static_cast<i64>(lev) * nf;
      for (int i = threadIdx.x; i < nf; i += blockDim.x) {
        T v = x0[i];
        if (i - s >= 0) v = v - c1[i] * x0[i - s];
        if (i + s < nf) v = v - c2[i] * x0[i + s];
        x1[i] = v;
      }
      __syncthreads();
      T* t = x0;
      x0 = x1;
      x1 = t;
    }
    SLAB_STAMP(3);
    for (int i = threadIdx.x; i < nf; i += blockDim.x)
      st_out(A.modes[a], static_cast<i64>(k) * nf + i, x0[i] * ld<T>(A.invb[a], static_cast<i64>(k) * nf + i));
#ifdef ASDSM_SLAB_TRACE
    __syncthreads();
    SLAB_STAMP(4);
    if (threadIdx.x == 0 && blockIdx.x == 0)
      printf("SLABDBG fwd a %d gather %lld stage %lld pcr %lld out %lld\n", a, T_[1] - T_[0], T_[2] - T_[1],
             T_[3] - T_[2], T_[4] - T_[3]);
#endif
    return;
  }
  constexpr int E = 6;  // elements per thread (line length <= 6144)
  T c1[E], c2[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = threadIdx.x + e * kThreads;
    const i64 base = static_cast<i64>(k) * L * nf;
    c1[e] = (i < nf && L > 0) ? ld<T>(K1, base + i) : zero_of<T>();
    c2[e] = (i < nf && L > 0) ? ld<T>(K2, base + i) : zero_of<T>();
  }
  int s = 1;
  for (int lev = 0; lev < L; ++lev, s <<= 1) {
    T n1[E], n2[E];
    const i64 nbase = (static_cast<i64>(k) * L + lev + 1) * nf;
#pragma unroll
    for (int e = 0; e < E; ++e) {  // prefetch the next level while this one computes
      const int i = threadIdx.x + e * kThreads;
      n1[e] = (i < nf && lev + 1 < L) ? ld<T>(K1, nbase + i) : zero_of<T>();
      n2[e] = (i < nf && lev + 1 < L) ? ld<T>(K2, nbase + i) : zero_of<T>();
    }
#pragma unroll
    for (int e = 0; e < E; ++e) {
      const int i = threadIdx.x + e * kThreads;
      if (i >= nf) break;
      T v = x0[i];
      if (i - s >= 0) v = v - c1[e] * x0[i - s];
      if (i + s < nf) v = v - c2[e] * x0[i + s];
      x1[i] = v;
    }
    __syncthreads();
    T* t = x0;
    x0 = x1;
    x1 = t;
#pragma unroll
    for (int e = 0; e < E; ++e) {
      c1[e] = n1[e];
      c2[e] = n2[e];
    }
  }
  for (int i = threadIdx.x; i < nf; i += blockDim.x)
    st_out(A.modes[a], static_cast<i64>(k) * nf + i, x0[i] * ld<T>(A.invb[a], static_cast<i64>(k) * nf + i));
}

template <typename T>
__global__ void __launch_bounds__(kRedThreads) slab2d_back_kernel(Slab2DArgs A, double* partials, DevState* S,
                                                                   double* history, CtrlArgs c, Skel2DArgs sk,
                                                                   int with_skel) {
  if (!S->active) return;
  SLAB_TRACE_DECL
  const MeshDev& m = A.m;
  double ss[2] = {0.0, 0.0};
  for (int a = 0; a < 2; ++a) {
    const int f = 1 - a, nc = m.nc[a], nf = m.nf[f];
    const i64 n = static_cast<i64>(nc) * nf;
    for (i64 t = static_cast<i64>(blockIdx.x) * blockDim.x + threadIdx.x; t < n; t += static_cast<i64>(gridDim.x) * blockDim.x) {
      int j, x;
      if (a == 0) {
        j = static_cast<int>(t % nc);
        x = static_cast<int>(t / nc);
      } else {
        x = static_cast<int>(t % nf);
        j = static_cast<int>(t / nf);
      }
      T acc = zero_of<T>();
      for (int k0 = 0; k0 < nc; k0 += 8) {
        T vv[8], mm[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int k = k0 + q;
          vv[q] = k < nc ? ld<T>(A.V[a], static_cast<i64>(j) * nc + k) : zero_of<T>();
          mm[q] = k < nc ? ld<T>(A.modes[a], static_cast<i64>(k) * nf + x) : zero_of<T>();
        }
#pragma unroll
        for (int q = 0; q < 8; ++q)
          if (k0 + q < nc) fma_acc(acc, vv[q], mm[q]);
      }
      const double v = real_part(acc);
      A.sol[a][t] = v;
      ss[a] += v * v;
    }
  }
  // partial sums: slot 0 = slab 0, slot 2 = slab 1
  __shared__ double sh[2][32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int q = 0; q < 2; ++q) {
    double v = ss[q];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sh[q][w] = v;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    for (int q = 0; q < 2; ++q) {
      double v = lane < nw ? sh[q][lane] : 0.0;
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      if (lane == 0) {
        partials[(2 * q) * kRedStride + blockIdx.x] = v;
        partials[(2 * q + 1) * kRedStride + blockIdx.x] = 0.0;
      }
    }
  }
  SLAB_STAMP(1);
  if (fold_ctrl(c, partials, S, history) && with_skel) {
    __syncthreads();
    SLAB_STAMP(2);
    if (S->have_e) skel2d_ccspline_block(sk);
#ifdef ASDSM_SLAB_TRACE
    __syncthreads();
    SLAB_STAMP(3);
    if (threadIdx.x == 0)
      printf("SLABDBG back blk %d compute %lld fold %lld ccspline %lld\n", blockIdx.x, T_[1] - T_[0], T_[2] - T_[1],
             T_[3] - T_[2]);
#endif
  }
}

}  // namespace

void slab2d_prepare() {
  static bool done = false;
  if (done) return;
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(slab2d_fwd_kernel<double>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(slab2d_fwd_kernel<cplx>, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmem));
  done = true;
}

void launch_slab2d_fwd(const Slab2DArgs& A, DevState* st, cudaStream_t s) {
  const int ncmax = std::max(A.m.nc[0], A.m.nc[1]);
  const int nfmax = std::max(A.m.nf[0], A.m.nf[1]);
  size_t smem = 2 * static_cast<size_t>(nfmax) * (A.cplx ? sizeof(cplx) : sizeof(double));
  const int lmax = std::max(A.levels[0], A.levels[1]);
  const size_t smem_full = smem + 2 * static_cast<size_t>(lmax) * nfmax * sizeof(double);
  Slab2DArgs B = A;
  B.pcr_smem = (!A.cplx && smem_full <= kSlabWOffset) ? 1 : 0;
  if (B.pcr_smem) smem = smem_full;
  if (smem > kSlabWOffset) throw AsdsmError(kUnsupported, "2D slab line longer than shared memory allows");
  smem = kMaxSmem;  // station weights sit at kSlabWOffset
  if (!A.cplx && nfmax > 6 * kThreads) throw AsdsmError(kUnsupported, "2D slab line longer than 6144");
  if (smem > kMaxSmem) throw AsdsmError(kUnsupported, "2D slab line longer than shared memory allows");
  dim3 grid(static_cast<unsigned>(ncmax), 2);
  if (A.cplx) slab2d_fwd_kernel<cplx><<<grid, kThreads, smem, s>>>(B, st);
  else slab2d_fwd_kernel<double><<<grid, kThreads, smem, s>>>(B, st);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void launch_slab2d_back(const Slab2DArgs& A, double* partials, DevState* st, double* history, bool with_norms,
                        cudaStream_t s, const Skel2DArgs* skel) {
  CtrlArgs c{};
  c.op = with_norms ? kCtrlSlabNorms2 : -1;
  Skel2DArgs sk{};
  if (skel) sk = *skel;
  const int ws = (skel && with_norms) ? 1 : 0;
  if (A.cplx) slab2d_back_kernel<cplx><<<kRedBlocks, kRedThreads, 0, s>>>(A, partials, st, history, c, sk, ws);
  else slab2d_back_kernel<double><<<kRedBlocks, kRedThreads, 0, s>>>(A, partials, st, history, c, sk, ws);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
