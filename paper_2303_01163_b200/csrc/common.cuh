// Shared device/host definitions for the ASDSM B200 library.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>

namespace asdsm_b200 {

using i64 = long long;

#define ASDSM_CUDA_CHECK(expr)                                                              \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      throw ::asdsm_b200::CudaError(std::string(#expr) + ": " + cudaGetErrorString(_e));   \
  } while (0)

struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// Complex arithmetic for mode spaces of operators whose 1D factor has complex eigenvalues
// (cell Peclet number > 2 on a coarse step).  Only the ops the solver needs.
struct cplx {
  double re, im;
};
#ifndef __CUDACC__
#ifndef __host__
#define __host__
#define __device__
#endif
#endif
__host__ __device__ inline cplx cmake(double r, double i) { return cplx{r, i}; }
__host__ __device__ inline cplx operator+(cplx a, cplx b) { return cplx{a.re + b.re, a.im + b.im}; }
__host__ __device__ inline cplx operator-(cplx a, cplx b) { return cplx{a.re - b.re, a.im - b.im}; }
__host__ __device__ inline cplx operator*(cplx a, cplx b) {
  return cplx{a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re};
}
__host__ __device__ inline cplx operator*(double a, cplx b) { return cplx{a * b.re, a * b.im}; }

template <typename T>
__host__ __device__ inline T zero_of();
template <>
__host__ __device__ inline double zero_of<double>() { return 0.0; }
template <>
__host__ __device__ inline cplx zero_of<cplx>() { return cplx{0.0, 0.0}; }

__host__ __device__ inline double real_part(double x) { return x; }
__host__ __device__ inline double real_part(cplx x) { return x.re; }
__host__ __device__ inline void fma_acc(double& acc, double a, double b) { acc = fma(a, b, acc); }
__host__ __device__ inline void fma_acc(cplx& acc, cplx a, cplx b) {
  acc.re = fma(a.re, b.re, acc.re);
  acc.re = fma(-a.im, b.im, acc.re);
  acc.im = fma(a.re, b.im, acc.im);
  acc.im = fma(a.im, b.re, acc.im);
}
__host__ __device__ inline void fma_acc(cplx& acc, double a, cplx b) {
  acc.re = fma(a, b.re, acc.re);
  acc.im = fma(a, b.im, acc.im);
}
__host__ __device__ inline void fma_acc(cplx& acc, cplx a, double b) {
  acc.re = fma(a.re, b, acc.re);
  acc.im = fma(a.im, b, acc.im);
}

// Non-contracted arithmetic: the residual/stencil kernels reproduce the reference's
// rounding sequence (CSR row dot in column order, proj/src/sparse.cpp:66-72) exactly.
#ifdef __CUDACC__
// Asynchronous global->shared copies (LDGSTS): many in flight per thread, no register staging.
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(s), "l"(gmem));
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
}
// Programmatic dependent launch: a kernel lets the next one in the stream start as soon as all of
// its CTAs are resident (launch_dependents), and the next one runs its data-independent prologue
// (table staging) before waiting for this grid's completion and memory (wait).  Both are no-ops
// for kernels launched without the attribute.
__device__ __forceinline__ void pdl_launch_dependents() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }
#endif

constexpr int kMaxDim = 3;

#ifdef __CUDACC__
// Launch with the programmatic-stream-serialization attribute (PDL; captured into the graph as a
// programmatic dependency) when ASDSM_PDL=1, plainly otherwise.
bool pdl_enabled();
template <typename... KArgs, typename... Args>
inline void launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  ASDSM_CUDA_CHECK(cudaLaunchKernelEx(&cfg, kernel, args...));
}
#endif

// Host-side count of kernels this library launched (reported as gpu_launches by bench.py).
extern long long g_kernel_launches;
constexpr int kNumSms = 148;

}  // namespace asdsm_b200
