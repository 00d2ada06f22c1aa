// One-launch 2D slab step (error mode, lines up to kPartMaxLine fine points).
//
// The reference solves the two anisotropic slab systems A_fc, A_cf with SparseLU
// (linsolve.cpp:58-66, solver.cpp:550-558), normalizes both solutions (solver.cpp:79-84),
// takes the cross values and clamped-spline corrections (solver.cpp:166-187, spline.cpp) and
// scatters the skeleton into the fine array.  Here a cluster of two CTAs does all of it in one
// launch, CTA a owning slab a (coarse along axis a):
//   P1  the residual on the slab's stations (compact copy kept by the residual passes), the
//       eigenvector blocks and the line-solve tables -> shared memory; every CTA of a slab
//       takes a quarter of the fine points (a cluster of 8 CTAs, four per slab)
//   P2  transform along the coarse axis on the DMMA pipe: nc mode lines of nf fine points
//   P3  one warp per mode line: partitioned tridiagonal solve -- every lane a Thomas sweep over
//       its SEG-row segment (in registers), a shuffle-PCR over the separators, the segment
//       reconstruction (tables: SepSolver::part) -- no block-wide barriers inside
//   P4  back transform to the slab layout (kept in shared memory) + squared norm
//   P5  norms and cross values exchanged through distributed shared memory
//   P6  cross-point corrections and spline segments (both families, redundantly per CTA)
//   P7  skeleton write: CTA 1 the lines along x (with the reference's cross-point rounding),
//       CTA 0 the lines along y
// Divisions by mesh constants and by the slab norms are reciprocal multiplies here (the
// reference divides): values agree to an ulp, far inside the 1e-10 parity tolerance.
#include "slabstep2d.cuh"
#include "partsolve.cuh"

#include <cooperative_groups.h>

namespace asdsm_b200 {

namespace cg = cooperative_groups;

namespace {

constexpr int kStepThreads = 256;
constexpr int kStepWarps = kStepThreads / 32;
constexpr int kStepMaxNc = 24;
#ifndef ASDSM_SLAB_CTAS
#define ASDSM_SLAB_CTAS 8
#endif
// CTAs per slab; the cluster is both slabs: 16 CTAs (a non-portable cluster size, checked with
// slabstep2d_launchable) -- measured, config 1: slab step 14.5 -> 12.6 us, solve -2.8 % against
// 4 per slab (ASDSM_SLAB_CTAS=4 at build time)
constexpr int kSlabCtas = ASDSM_SLAB_CTAS;
constexpr int kClusterCtas = 2 * kSlabCtas;
constexpr int kOwnMax = (kStepMaxNc + kSlabCtas - 1) / kSlabCtas;  // mode lines one CTA solves

struct StepLayout {
  int NC, XR, NF, PS;
  int st, md, ml, wv, pt, cr1, cr2, nrm, ce1, ce2, red, total;
};

// x-range of part c of a line of n points
__host__ __device__ inline int xr_begin(int n, int c) { return (n * c) / kSlabCtas; }

__host__ __device__ inline StepLayout step_layout(const MeshDev& m, int pstride) {
  StepLayout L{};
  L.NC = m.nc[0] > m.nc[1] ? m.nc[0] : m.nc[1];
  L.NF = m.nf[0] > m.nf[1] ? m.nf[0] : m.nf[1];
  L.XR = (L.NF + kSlabCtas - 1) / kSlabCtas + 1;
  L.PS = pstride;
  const int ncc = m.nc[0] * m.nc[1];
  int o = 0;
  auto take = [&](int n) {
    const int r = o;
    o += (n + 1) & ~1;  // keep 16-byte alignment of every region
    return r;
  };
  L.st = take(L.NC * L.XR);          // stations of this x-range, then the slab solution there
  L.md = take(L.NC * L.XR);          // modes of this x-range
  L.ml = take(kOwnMax * L.NF);       // full mode lines this CTA solves
  L.wv = take(2 * L.NC * L.NC);
  L.pt = take(kOwnMax * pstride);
  L.cr1 = take(ncc);
  L.cr2 = take(ncc);
  L.nrm = take(kClusterCtas);
  L.ce1 = take(ncc);
  L.ce2 = take(ncc);
  L.red = take(32);
  L.total = o;
  return L;
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// C[nc][ld] = Amat[nc][nc] * B[nc][ld] over the first nx columns (B, C in shared memory;
// MT = ceil(nc/8) row tiles, KS = ceil(nc/4) k steps of m8n8k4), warps over 8-column tiles;
// returns the warp's sum of squares of C when kNorm.
template <int MT, int KS, bool kNorm>
__device__ __forceinline__ double small_gemm(const double* Amat, const double* B, double* C, int nc, int nx, int ld) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, r8 = lane >> 2, c4 = lane & 3;
  double a[MT][KS];
#pragma unroll
  for (int mt = 0; mt < MT; ++mt)
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int row = mt * 8 + r8, k = ks * 4 + c4;
      a[mt][ks] = (row < nc && k < nc) ? Amat[row * nc + k] : 0.0;
    }
  double ss = 0.0;
  const int ntiles = (nx + 7) >> 3;
  for (int nt = warp; nt < ntiles; nt += kStepWarps) {
    const int n0 = nt * 8;
    double b[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = ks * 4 + c4;
      b[ks] = (k < nc && n0 + r8 < nx) ? B[k * ld + n0 + r8] : 0.0;
    }
    double acc[MT][2];
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) acc[mt][0] = acc[mt][1] = 0.0;
#pragma unroll
    for (int ks = 0; ks < KS; ++ks)
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) dmma884(acc[mt], a[mt][ks], b[ks]);
#pragma unroll
    for (int mt = 0; mt < MT; ++mt) {
      const int row = mt * 8 + r8;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = n0 + 2 * c4 + h;
        if (row < nc && col < nx) {
          C[row * ld + col] = acc[mt][h];
          if (kNorm) ss += acc[mt][h] * acc[mt][h];
        }
      }
    }
  }
  return ss;
}

template <bool kNorm>
__device__ __forceinline__ double gemm_dispatch(const double* Amat, const double* B, double* C, int nc, int nx, int ld) {
  if (nc <= 4) return small_gemm<1, 1, kNorm>(Amat, B, C, nc, nx, ld);
  if (nc <= 8) return small_gemm<1, 2, kNorm>(Amat, B, C, nc, nx, ld);
  if (nc <= 12) return small_gemm<2, 3, kNorm>(Amat, B, C, nc, nx, ld);
  if (nc <= 16) return small_gemm<2, 4, kNorm>(Amat, B, C, nc, nx, ld);
  if (nc <= 20) return small_gemm<3, 5, kNorm>(Amat, B, C, nc, nx, ld);
  return small_gemm<3, 6, kNorm>(Amat, B, C, nc, nx, ld);
}

// Cluster of 2 x kSlabCtas CTAs: CTA (a, c) owns slab a's fine x-range c (stations, transforms,
// solution, skeleton write) and the mode lines k = c, c + kSlabCtas, ... (line solves); the
// mode lines move between the two ownerships through distributed shared memory.
template <int SEG>
__global__ void __cluster_dims__(kClusterCtas, 1, 1) __launch_bounds__(kStepThreads, 1)
    slabstep2d_kernel(SlabStep2DArgs A, DevState* S) {
  pdl_launch_dependents();
#ifdef ASDSM_STEP_TRACE
  long long T_[12] = {clock64(), 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define STEP_STAMP(i) T_[i] = clock64()
#else
#define STEP_STAMP(i)
#endif
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double sm[];
  const MeshDev& m = A.m;
  const int PS = A.pstride[0] > A.pstride[1] ? A.pstride[0] : A.pstride[1];
  const StepLayout Lo = step_layout(m, PS);
  const int rank = static_cast<int>(cluster.block_rank());
  const int a = rank / kSlabCtas, c = rank % kSlabCtas;
  const int nc = m.nc[a], nf = m.nf[1 - a];
  const int x0 = xr_begin(nf, c), nx = xr_begin(nf, c + 1) - x0, XR = Lo.XR;
  const int nc0 = m.nc[0], nc1 = m.nc[1], ncc = nc0 * nc1;
  const int nown = (nc - c + kSlabCtas - 1) / kSlabCtas;  // modes c, c + C, ... < nc
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* st = sm + Lo.st;
  double* md = sm + Lo.md;
  double* ml = sm + Lo.ml;
  double* sW = sm + Lo.wv;
  double* sV = sW + nc * nc;
  double* pt = sm + Lo.pt;
  // P1: the eigenvector blocks, the owned modes' line tables and the spline basis (constant:
  // staged while the previous kernel drains), then this x-range of the stations
  for (int i = tid; i < nc * nc; i += kStepThreads) {
    cp_async8(sW + i, A.W[a] + i);
    cp_async8(sV + i, A.V[a] + i);
  }
  for (int i = tid; i < nown * A.pstride[a]; i += kStepThreads) {
    const int u = i / A.pstride[a], o = i - u * A.pstride[a];
    cp_async8(pt + u * PS + o, A.part[a] + static_cast<i64>(c + u * kSlabCtas) * A.pstride[a] + o);
  }
  pdl_wait();
  if (!S->active) {  // same decision in every CTA of the cluster
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;\n" ::: "memory");
    return;
  }
  const double* rs = (S->cur ? A.sta1 : A.sta0) + (a == 0 ? 0 : static_cast<i64>(nc0) * m.nf[1]);
  for (int i = tid; i < nc * nx; i += kStepThreads) {
    const int j = i / nx, x = i - j * nx;
    cp_async8(st + j * XR + x, rs + static_cast<i64>(j) * nf + x0 + x);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  STEP_STAMP(1);
  // P2: md = W st on this x-range, then every mode row to its owner's full line (DSMEM)
  gemm_dispatch<false>(sW, st, md, nc, nx, XR);
  __syncthreads();
  for (int i = tid; i < nc * nx; i += kStepThreads) {
    const int k = i / nx, x = i - k * nx;
    double* dst = cluster.map_shared_rank(ml, a * kSlabCtas + k % kSlabCtas);
    dst[(k / kSlabCtas) * Lo.NF + x0 + x] = md[k * XR + x];
  }
  cluster.sync();
  STEP_STAMP(2);
  // P3: one warp per owned mode line
  if (warp < nown) {
    const int k = c + warp * kSlabCtas;
    (void)k;
    part_solve_line<SEG>(ml + warp * Lo.NF, pt + warp * PS, nf, A.pP[a], A.plast[a], A.line_l[a], A.line_r[a]);
  }
  STEP_STAMP(10);
  cluster.sync();
  STEP_STAMP(3);
  // P4: pull this x-range of every mode line back, sol = V md, squared norm
  for (int i = tid; i < nc * nx; i += kStepThreads) {
    const int k = i / nx, x = i - k * nx;
    const double* src = cluster.map_shared_rank(ml, a * kSlabCtas + k % kSlabCtas);
    md[k * XR + x] = src[(k / kSlabCtas) * Lo.NF + x0 + x];
  }
  __syncthreads();
  double ss = gemm_dispatch<true>(sV, md, st, nc, nx, XR);
  double* red = sm + Lo.red;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, o);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  STEP_STAMP(4);
  // P5: norms (per-CTA partials to every CTA, summed in rank order) and cross values
  double* nrm = sm + Lo.nrm;
  double* cr1 = sm + Lo.cr1;  // u_fc at the cross points (slab 1)
  double* cr2 = sm + Lo.cr2;  // u_cf at the cross points (slab 0)
  if (tid < kClusterCtas) {
    double t = 0.0;
    for (int w = 0; w < kStepWarps; ++w) t += red[w];
    cluster.map_shared_rank(nrm, tid)[rank] = t;
  }
  for (int t = tid; t < ncc * kClusterCtas; t += kStepThreads) {
    const int dst = t / ncc, q = t - dst * ncc;
    const int I = q % nc0, J = q / nc0;
    const int x = a == 1 ? (I + 1) * m.n[0] - 1 : (J + 1) * m.n[1] - 1;  // along this slab's fine axis
    if (x < x0 || x >= x0 + nx) continue;
    const double v = a == 1 ? st[J * XR + x - x0] : st[I * XR + x - x0];
    cluster.map_shared_rank(a == 1 ? cr1 : cr2, dst)[q] = v;
  }
  cluster.sync();
  STEP_STAMP(5);
  double s0 = 0.0, s1 = 0.0;
  for (int r = 0; r < kSlabCtas; ++r) {
    s0 += nrm[r];
    s1 += nrm[kSlabCtas + r];
  }
  const double ncf = sqrt(s0), nfc = sqrt(s1);
  if (rank == 0 && tid == 0) {
    S->slab_norm[0] = ncf;
    S->slab_norm[1] = nfc;
    if (!(ncf > 0.0) || !(nfc > 0.0)) S->have_e = 0;
  }
  if (!(ncf > 0.0) || !(nfc > 0.0)) return;  // ZeroNormSolution: no correction this step
  const double ifc = 1.0 / nfc, icf = 1.0 / ncf;
  STEP_STAMP(9);
  // P6: corrections at the cross points (error mode: the coin picks the slab)
  double* ce1 = sm + Lo.ce1;
  double* ce2 = sm + Lo.ce2;
  const bool take_fc = A.coin[0] != 0;
  for (int t = tid; t < ncc; t += kStepThreads) {
    const double u1 = cr1[t] * ifc, u2 = cr2[t] * icf;
    const double uh = take_fc ? u1 : u2;
    ce1[t] = __dsub_rn(uh, u1);
    ce2[t] = __dsub_rn(uh, u2);
  }
  __syncthreads();
  STEP_STAMP(8);
  STEP_STAMP(6);
  // P7: publish what the skeleton is made of -- the normalized slab values on this x-range of
  // every station line, the cross-point corrections and the cross points themselves.  The hole
  // kernel evaluates its ring from these (value / norm + spline of the corrections) and writes
  // the skeleton lines it owns, so the line values are computed by 100 CTAs instead of 8.
  {
    const double inv = a == 1 ? ifc : icf;
    double* dst = (a == 1 ? A.skel_line1 : A.skel_line0) + x0;
    for (int j = 0; j < nc; ++j)
      for (int x = tid; x < nx; x += kStepThreads) dst[static_cast<i64>(j) * nf + x] = st[j * XR + x] * inv;
    if (rank == 0) {
      const i64 Nx = m.nf[0];
      for (int t = tid; t < ncc; t += kStepThreads) {
        A.corr[t] = ce1[t];
        A.corr[ncc + t] = ce2[t];
        // cross point (reference merge order: lines along x, then the y-line value added and
        // removed): av = P(u_fc)/nfc + E1 (B is the identity at knots), bv = P(u_cf)/ncf + E2
        const int I = t % nc0, J = t / nc0;
        const double av = __dadd_rn(cr1[t] * ifc, ce1[t]);
        const double bv = __dadd_rn(cr2[t] * icf, ce2[t]);
        A.out[(I + 1) * m.n[0] - 1 + Nx * ((J + 1) * m.n[1] - 1)] = __dadd_rn(__dadd_rn(av, bv), -bv);
      }
    }
  }
#ifdef ASDSM_STEP_TRACE
  __syncthreads();
  STEP_STAMP(7);
  if (tid == 0 && (rank == 0 || rank == kSlabCtas))
    printf("STEPDBG cta %d load %lld tf+scatter %lld solve %lld (own %lld) back %lld xchg %lld norm %lld corr %lld write %lld\n",
           rank, T_[1] - T_[0], T_[2] - T_[1], T_[3] - T_[2], T_[10] - T_[2], T_[4] - T_[3], T_[5] - T_[4], T_[9] - T_[5],
           T_[8] - T_[9], T_[7] - T_[6]);
#endif
#undef STEP_STAMP
}

}  // namespace

bool slabstep2d_supported(const MeshDev& m, const SepSolver* slab) {
  if (m.dim != 2 || m.nc[0] > kStepMaxNc - 2 || m.nc[1] > kStepMaxNc - 2) return false;
  for (int a = 0; a < 2; ++a)
    if (slab[a].part == nullptr || slab[a].complex_modes) return false;
  if (slab[0].part_seg != slab[1].part_seg) return false;
  const int ps = std::max(slab[0].part_stride, slab[1].part_stride);
  return sizeof(double) * static_cast<size_t>(step_layout(m, ps).total) <= 220 * 1024;
}

size_t slabstep2d_smem_bytes(const SlabStep2DArgs& A) {
  return sizeof(double) * static_cast<size_t>(step_layout(A.m, std::max(A.pstride[0], A.pstride[1])).total);
}

// one kernel per segment length: a single solve body per kernel keeps the code small enough
// to stay resident (measured: with every length behind one switch the line solve ran 5x slower)
#define ASDSM_FOR_SEGS(X) X(2) X(4) X(8) X(12) X(16) X(20) X(24) X(28) X(32)

void slabstep2d_prepare() {
#define ASDSM_SEG_ATTR(S_)                                                                                 \
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(slabstep2d_kernel<S_>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                        220 * 1024));                                                      \
  if (kClusterCtas > 8)                                                                                     \
    ASDSM_CUDA_CHECK(cudaFuncSetAttribute(slabstep2d_kernel<S_>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  ASDSM_FOR_SEGS(ASDSM_SEG_ATTR)
#undef ASDSM_SEG_ATTR
}

bool slabstep2d_launchable(const SlabStep2DArgs& A) {
  if (A.pseg[0] != A.pseg[1]) return false;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kClusterCtas);
  cfg.blockDim = dim3(kStepThreads);
  cfg.dynamicSmemBytes = slabstep2d_smem_bytes(A);
  int n = 0;
  cudaError_t e = cudaErrorInvalidValue;
  switch (A.pseg[0]) {
#define ASDSM_SEG_OCC(S_) \
  case S_:                \
    e = cudaOccupancyMaxActiveClusters(&n, slabstep2d_kernel<S_>, &cfg); \
    break;
    ASDSM_FOR_SEGS(ASDSM_SEG_OCC)
#undef ASDSM_SEG_OCC
    default:
      break;
  }
  if (e != cudaSuccess) {
    cudaGetLastError();  // clear: the caller falls back to the three-launch slab path
    return false;
  }
  return n > 0;
}

void launch_slabstep2d(const SlabStep2DArgs& A, DevState* st, cudaStream_t s) {
  if (A.pseg[0] != A.pseg[1]) throw AsdsmError(kUnsupported, "slab step: slabs with different segment lengths");
  const size_t smem = slabstep2d_smem_bytes(A);
  switch (A.pseg[0]) {
#define ASDSM_SEG_LAUNCH(S_) \
  case S_:                   \
    launch_pdl(slabstep2d_kernel<S_>, kClusterCtas, kStepThreads, smem, s, A, st); \
    break;
    ASDSM_FOR_SEGS(ASDSM_SEG_LAUNCH)
#undef ASDSM_SEG_LAUNCH
    default:
      throw AsdsmError(kUnsupported, "slab step: unsupported segment length");
  }
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
