// Probe: TMA 2D box loads of a pair-row view (2 N_x, N_y N_z / 2) of an odd-row-length array.
// nvcc -gencode arch=compute_100a,code=sm_100a -o probe_tma_pairs probe_tma_pairs.cu
// ./probe_tma_pairs VARIANT  (bit 0: tensor map in global memory; bit 1: shared::cta destination;
// bit 2: UINT64 element type; bit 3: no L2 promotion; bit 4: no .tile qualifier)
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>

__device__ __forceinline__ unsigned smem_u32(const void* p) { return static_cast<unsigned>(__cvta_generic_to_shared(p)); }

template <int V>
__global__ void probe(const __grid_constant__ CUtensorMap m, const CUtensorMap* gm, int c0, int c1, int txb, double* out) {
  extern __shared__ __align__(128) double raw[];
  double* sm = reinterpret_cast<double*>((reinterpret_cast<uintptr_t>(raw) + 127) & ~uintptr_t(127));
  __shared__ __align__(8) unsigned long long bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar)), "r"(1) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long desc = (V & 1) ? reinterpret_cast<unsigned long long>(gm) : reinterpret_cast<unsigned long long>(&m);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)), "r"(txb * 10 * 8) : "memory");
    if (V & 2)
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(sm)),
                   "l"(desc), "r"(c0), "r"(c1), "r"(smem_u32(&bar)) : "memory");
    else if (V & 16)
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(sm)),
                   "l"(desc), "r"(c0), "r"(c1), "r"(smem_u32(&bar)) : "memory");
    else
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(sm)),
                   "l"(desc), "r"(c0), "r"(c1), "r"(smem_u32(&bar)) : "memory");
  }
  unsigned done = 0;
  while (!done) {
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(smem_u32(&bar)), "r"(0) : "memory");
  }
  for (int i = threadIdx.x; i < txb * 10; i += blockDim.x) out[i] = sm[i];
}

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                                 const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                 CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

template <int V>
void launch(const CUtensorMap& m, const CUtensorMap* gm, int c0, int c1, int txb, double* out) {
  probe<V><<<1, 128, 128 + txb * 10 * 8 + 256>>>(m, gm, c0, c1, txb, out);
}

int main(int argc, char** argv) {
  const int V = argc > 1 ? atoi(argv[1]) : 0;
  void* p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeTiled enc = reinterpret_cast<EncodeTiled>(p);
  const int shapes[3][3] = {{128, 2, 128}, {24, 24, 24}, {509, 509, 9}};
  int bad = 0;
  for (int si = 0; si < 3; ++si) {
    const int Nx = shapes[si][0], Ny = shapes[si][1], Nz = shapes[si][2];
    const long long n = 1LL * Nx * Ny * Nz;
    std::vector<double> h(n + Nx + 2);
    for (long long i = 0; i < n; ++i) h[i] = double(i);
    double *d, *out;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    cudaMalloc(&out, 4096 * 8);
    const int TX = Nx < 128 ? Nx : 128;
    const int txb = si == 0 ? 32 : ((TX + 3) & ~1);
    CUtensorMap m;
    memset(&m, 0, sizeof(m));
    cuuint64_t dims[2] = {cuuint64_t(2 * Nx), cuuint64_t((1LL * Ny * Nz + 1) / 2)};
    cuuint64_t strides[1] = {cuuint64_t(2 * Nx) * 8};
    cuuint32_t box[2] = {cuuint32_t(txb), 10};
    cuuint32_t es[2] = {1, 1};
    CUresult r = enc(&m, (V & 4) ? CU_TENSOR_MAP_DATA_TYPE_UINT64 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                     (V & 8) ? CU_TENSOR_MAP_L2_PROMOTION_NONE : CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    CUtensorMap* gm = nullptr;
    cudaMalloc(&gm, sizeof(CUtensorMap));
    cudaMemcpy(gm, &m, sizeof(m), cudaMemcpyHostToDevice);
    printf("variant %d shape %d %d %d encode %d\n", V, Nx, Ny, Nz, int(r));
    const int cs[3][2] = {{0, 0}, {Nx - 1, 3}, {-1, -1}};
    for (auto& c : cs) {
      switch (V & 3) {
        case 0: (V & 16) ? launch<16>(m, gm, c[0], c[1], txb, out) : launch<0>(m, gm, c[0], c[1], txb, out); break;
        case 1: launch<1>(m, gm, c[0], c[1], txb, out); break;
        case 2: launch<2>(m, gm, c[0], c[1], txb, out); break;
        default: launch<3>(m, gm, c[0], c[1], txb, out); break;
      }
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) {
        printf("variant %d coords (%d,%d): %s\n", V, c[0], c[1], cudaGetErrorString(e));
        return 1;
      }
      std::vector<double> o(txb * 10);
      cudaMemcpy(o.data(), out, o.size() * 8, cudaMemcpyDeviceToHost);
      int errs = 0;
      for (int j = 0; j < 10; ++j)
        for (int i = 0; i < txb; ++i) {
          const long long x = c[0] + i, pj = c[1] + j;
          double want = 0.0;
          if (x >= 0 && x < 2 * Nx && pj >= 0 && pj < (long long)dims[1]) want = h[pj * 2 * Nx + x];
          if (o[j * txb + i] != want) ++errs;
        }
      printf("variant %d coords (%d,%d): %d mismatches\n", V, c[0], c[1], errs);
      bad += errs;
    }
  }
  printf(bad ? "FAIL\n" : "OK\n");
  return bad != 0;
}
