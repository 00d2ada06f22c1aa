// DMMA (fp64 tensor-pipe mma.sync) transform GEMM for sm_100a.  Same FP64 peak as DFMA on
// B200 (both ~37 TFLOP/s measured), but each 8x8x4 MMA takes one A and one B operand
// per lane, so a 32x32 warp tile needs 8 shared-memory loads per 16 MMAs (4096 FMAs) --
// the scalar register-tiled kernel is limited by shared-memory bandwidth instead.
#include "dmma_gemm.cuh"

namespace asdsm_b200 {

namespace {

constexpr int BP = 64, BQ = 64, BK = 32, PAD = 4, NTH = 128;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void line_base(const GemmLines& L, i64 p, i64& ib, i64& ob) {
  const i64 o0 = p % L.o_ext[0];
  i64 t = p / L.o_ext[0];
  const i64 o1 = t % L.o_ext[1];
  t /= L.o_ext[1];
  const i64 h0 = t % L.nbox[0];
  t /= L.nbox[0];
  const i64 h1 = t % L.nbox[1];
  const i64 h2 = t / L.nbox[1];
  ib = h0 * L.in_bs[0] + h1 * L.in_bs[1] + h2 * L.in_bs[2] + o0 * L.o_in[0] + o1 * L.o_in[1];
  ob = h0 * L.out_bs[0] + h1 * L.out_bs[1] + h2 * L.out_bs[2] + o0 * L.o_out[0] + o1 * L.o_out[1];
}

template <bool kContigIn, bool kContigOut>
__global__ void __launch_bounds__(NTH) dmma_transform_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                             const double* __restrict__ M, int m, i64 in_es, i64 out_es,
                                                             GemmLines L) {
  __shared__ double As[BP][BK + PAD];
  __shared__ double Bs[BQ][BK + PAD];
  __shared__ i64 s_ib[BP], s_ob[BP];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const i64 p0 = static_cast<i64>(blockIdx.y) * BP;  // grid = (q tiles, line blocks)
  const int q0 = blockIdx.x * BQ;
  if (tid < BP) {
    i64 ib = 0, ob = 0;
    if (p0 + tid < L.nlines) line_base(L, p0 + tid, ib, ob);
    s_ib[tid] = ib;
    s_ob[tid] = ob;
  }
  __syncthreads();
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int wp = (warp >> 1) * 32, wq = (warp & 1) * 32;
  constexpr int PER = (BP * BK) / NTH;  // 16
  double ra[PER], rb[PER];
  auto load = [&](int k0) {
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int e = tid + r * NTH;
      int pl, kl;
      if (kContigIn) {
        pl = e / BK;
        kl = e % BK;
      } else {
        pl = e % BP;
        kl = e / BP;
      }
      const int k = k0 + kl;
      ra[r] = (p0 + pl < L.nlines && k < m) ? __ldg(in + s_ib[pl] + static_cast<i64>(k) * in_es) : 0.0;
      const int ql = e / BK, kq = e % BK;
      rb[r] = (q0 + ql < m && k0 + kq < m) ? __ldg(M + static_cast<i64>(q0 + ql) * m + k0 + kq) : 0.0;
    }
  };
  auto store = [&]() {
#pragma unroll
    for (int r = 0; r < PER; ++r) {
      const int e = tid + r * NTH;
      if (kContigIn) As[e / BK][e % BK] = ra[r];
      else As[e % BP][e / BP] = ra[r];
      Bs[e / BK][e % BK] = rb[r];
    }
  };
  load(0);
  for (int k0 = 0; k0 < m; k0 += BK) {
    store();
    __syncthreads();
    if (k0 + BK < m) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[wp + i * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[wq + j * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int pl = wp + i * 8 + (lane >> 2);
    if (p0 + pl >= L.nlines) continue;
    const i64 ob = s_ob[pl];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int q = q0 + wq + j * 8 + 2 * (lane & 3);
      if (kContigOut && q + 1 < m) {
        double* dst = out + ob + q;
        if ((reinterpret_cast<uintptr_t>(dst) & 15) == 0) {
          *reinterpret_cast<double2*>(dst) = make_double2(acc[i][j][0], acc[i][j][1]);
        } else {
          dst[0] = acc[i][j][0];
          dst[1] = acc[i][j][1];
        }
      } else {
        if (q < m) out[ob + static_cast<i64>(q) * out_es] = acc[i][j][0];
        if (q + 1 < m) out[ob + static_cast<i64>(q + 1) * out_es] = acc[i][j][1];
      }
    }
  }
}

}  // namespace

void dmma_prepare() {}  // the register-staged kernel needs no attributes (a 3-stage cp.async
                        // variant measured slower on both m=102 and m=409 and was dropped)

void launch_dmma_transform(const double* in, double* out, const double* M, int m, i64 in_es, i64 out_es,
                           const GemmLines& L, cudaStream_t s) {
  // q tiles fastest: the CTAs re-reading the same A rows are co-scheduled (L2 hits)
  const i64 pb = (L.nlines + BP - 1) / BP;
  const unsigned qb = static_cast<unsigned>((m + BQ - 1) / BQ);
  if (pb > 65535) throw AsdsmError(kUnsupported, "transform batch too large for the grid");
  dim3 grid(qb, static_cast<unsigned>(pb));
  const bool ci = in_es == 1, co = out_es == 1;
  if (ci && co) dmma_transform_kernel<true, true><<<grid, NTH, 0, s>>>(in, out, M, m, in_es, out_es, L);
  else if (ci) dmma_transform_kernel<true, false><<<grid, NTH, 0, s>>>(in, out, M, m, in_es, out_es, L);
  else if (co) dmma_transform_kernel<false, true><<<grid, NTH, 0, s>>>(in, out, M, m, in_es, out_es, L);
  else dmma_transform_kernel<false, false><<<grid, NTH, 0, s>>>(in, out, M, m, in_es, out_es, L);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
