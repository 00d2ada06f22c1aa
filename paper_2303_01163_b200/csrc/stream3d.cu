// 3D fine-grid pass with TMA-staged planes (north-star kernels 1 and 4, 3D):
//   UPDATE   : v = u + s e ; u' = v ; r' = b - A v         (solver.cpp:634-645, fdm.cpp:221-230)
//   RESIDUAL : v = u ; r = b - A v
// plus the norms (res_l2, res_inf, err) as block partials folded into the control op.
//
// One CTA per SM walks a contiguous share of the flattened (x-y tile, z) space, so every SM
// gets the same number of planes whatever the mesh; a tile is TX x 16 points (TX <= 128, a
// balanced split of the x extent) and is marched in z.
//
// TMA with odd row lengths: the fine arrays keep the reference's layout (x fastest, N_x odd), so
// no tensor map can describe them as (x, y, z) -- every global stride of a tensor map must be a
// multiple of 16 bytes.  Viewed as rows of PAIRS of grid rows, (2 N_x, N_y N_z / 2), the one
// stride is 16 N_x bytes: a tile's rows of one plane are two 2D boxes, the even rows and the odd
// rows (box x origins rounded down to a 16-byte boundary, as the TMA unit requires;
// out-of-range boxes are zero-filled; values read across a row end are never used).
//
// Warp-specialized, no CTA barrier in the loop: a producer warp issues, per plane step q, the
// u and e boxes of plane q (18 rows: the tile and its y halo) and the b (and exact) boxes of
// plane q - 1 into one stage of a 2-3 deep mbarrier ring; 16 consumer warps (4 column groups of
// 32 x 4 row groups of 4) each own 32 columns x 4 rows and march z with the three v planes in
// registers: per step a lane forms v = u + s e of plane q on its column for its 4 rows, the two
// y-halo rows and (lanes 0 / 31) the neighbouring column, takes the x neighbours from its
// neighbour lanes by shuffles, writes r and u' of plane q - 1, and releases the stage.  Each v
// costs one read of u and e, so the pass moves u, e, b in and u', r out -- 40 B per point (+8
// with an exact solution) plus the y-halo rows neighbouring tiles re-read from L2.  The row sum
// keeps the reference's CSR column order (fdm.cpp:110-117) with non-contracted arithmetic, so r
// is bitwise the two-pass (axpy + residual) result.
#include "ctrl.cuh"
#include "march.cuh"

#include <cuda.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

namespace asdsm_b200 {

namespace {

constexpr int kS3Warps = 16;                      // consumer warps
constexpr int kS3Cons = kS3Warps * 32;
constexpr int kS3Threads = kS3Cons + 32;          // + one producer warp
constexpr int kS3CG = 4, kS3RG = 4;               // column groups (32 columns), row groups
constexpr int kS3R = 4;                           // rows per consumer thread
constexpr int kS3TY = kS3RG * kS3R;               // tile rows (16)
constexpr int kS3MaxTX = kS3CG * 32;              // 128
constexpr int kS3PairsUE = (kS3TY + 2) / 2 + 1;   // u/e: 18 rows from any parity -> 10 pairs
constexpr int kS3PairsB = kS3TY / 2 + 1;          // b / exact: 16 rows -> 9 pairs
constexpr int kS3MaxStages = 3;

struct S3Geo {
  int tx, ntx, nty;  // tile width, tiles along x / y
  int txb;           // box width (doubles): TX + 3 rounded up to even
  int box_ue, box_b; // doubles per box in shared memory (128-byte multiples)
  long long work;    // ntx * nty * Nz planes
  int ns;            // pipeline stages
};

struct S3Maps {  // tensor maps of the pair-row views
  CUtensorMap u0, u1, e, b, x;
};

__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned long long* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(unsigned long long* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(unsigned long long* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned long long* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1, unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
          smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// The sequence of plane steps one CTA walks: its share [w0, w1) of the flattened (tile, z)
// space as per-tile segments [zb, ze); a segment takes steps q = zb-1 .. ze.  Producer and
// consumers walk identical copies.
struct PlaneSeq {
  long long w, w1;
  int nz;
  int tile, zb, ze, q;
  bool valid;
  __device__ void start(long long w0_, long long w1_, int nz_) {
    w = w0_;
    w1 = w1_;
    nz = nz_;
    next_segment();
  }
  __device__ void next_segment() {
    valid = w < w1;
    if (!valid) return;
    tile = static_cast<int>(w / nz);
    zb = static_cast<int>(w - static_cast<long long>(tile) * nz);
    const long long tend = static_cast<long long>(tile + 1) * nz;
    const long long end = w1 < tend ? w1 : tend;
    ze = static_cast<int>(end - static_cast<long long>(tile) * nz);
    w = end;
    q = zb - 1;
  }
  __device__ void advance() {
    if (++q > ze) next_segment();
  }
};

// first pair of the box holding rows [row, ...) of the pair view (row may be -1)
__device__ __forceinline__ int pair_of(long long row) { return static_cast<int>(row >= 0 ? row >> 1 : -1); }

template <bool UPD, bool EXACT>
__global__ void __launch_bounds__(kS3Threads, 1)
    stream3d_kernel(MarchArgs A, S3Geo G, const __grid_constant__ S3Maps M) {
  DevState* S = A.state;
  if (!S->active) return;
  const int cur = S->cur;
  double s = 0.0;
  bool work = true;
  if (UPD) {
    s = S->s;
    work = s != 0.0 && (!A.retry_pass || S->retry);
  }
  const int Nx = A.g.ext[0], Ny = A.g.ext[1], Nz = A.g.ext[2];
  const i64 sxy = A.g.stride[2];
  const int TX = G.tx, TXB = G.txb, BUE = G.box_ue, BB = G.box_b, NS = G.ns;
  constexpr int NUE = UPD ? 4 : 2;           // u (and e) boxes: even / odd rows
  constexpr int NB = EXACT ? 4 : 2;          // b (and exact) boxes
  const int SST = NUE * BUE + NB * BB;       // doubles per stage

  extern __shared__ __align__(128) double smem_raw[];
  // TMA destinations 128-byte aligned (an integer offset keeps the accesses in shared space)
  double* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u) / sizeof(double);
  __shared__ __align__(8) unsigned long long full[kS3MaxStages], empty[kS3MaxStages];

  const int tid = threadIdx.x;
  const long long w0 = G.work * blockIdx.x / gridDim.x, w1 = G.work * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], kS3Warps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (work && w0 < w1) {
    if (tid >= kS3Cons) {
      // ---- producer warp (lane 0 issues; the warp walks the loop together)
      const bool leader = tid == kS3Cons;
      PlaneSeq prod;
      prod.start(w0, w1, Nz);
      for (long long L = 0; prod.valid; ++L, prod.advance()) {
        const int stg = static_cast<int>(L % NS);
        if (L >= NS) mbar_wait(&empty[stg], static_cast<unsigned>(((L / NS) - 1) & 1));
        if (leader) {
          const int q = prod.q;
          const int x0 = (prod.tile % G.ntx) * TX, y0 = (prod.tile / G.ntx) * kS3TY;
          const bool ue = q >= 0 && q < Nz;
          const bool bq = q - 1 >= prod.zb && q - 1 < prod.ze;
          const unsigned bytes = (ue ? NUE * kS3PairsUE * TXB * 8u : 0u) + (bq ? NB * kS3PairsB * TXB * 8u : 0u);
          double* d = smem + static_cast<size_t>(stg) * SST;
          const int ce = (x0 - 1) & ~1, co = (Nx + x0 - 1) & ~1;  // 16-byte aligned box origins
          if (bytes) mbar_arrive_expect_tx(&full[stg], bytes);
          else mbar_arrive(&full[stg]);
          if (ue) {
            const int j0 = pair_of(static_cast<long long>(y0 - 1) + static_cast<long long>(q) * Ny);
            // (the buffer is picked by a branch, not a pointer select: the tensor map operand
            // must stay a kernel-parameter address, never a local copy)
            if (cur) {
              tma_load_2d(d, &M.u1, ce, j0, &full[stg]);
              tma_load_2d(d + BUE, &M.u1, co, j0, &full[stg]);
            } else {
              tma_load_2d(d, &M.u0, ce, j0, &full[stg]);
              tma_load_2d(d + BUE, &M.u0, co, j0, &full[stg]);
            }
            if (UPD) {
              tma_load_2d(d + 2 * BUE, &M.e, ce, j0, &full[stg]);
              tma_load_2d(d + 3 * BUE, &M.e, co, j0, &full[stg]);
            }
          }
          if (bq) {
            const int jb = pair_of(static_cast<long long>(y0) + static_cast<long long>(q - 1) * Ny);
            const int cb = x0 & ~1, cbo = (Nx + x0) & ~1;
            double* db = d + NUE * BUE;
            tma_load_2d(db, &M.b, cb, jb, &full[stg]);
            tma_load_2d(db + BB, &M.b, cbo, jb, &full[stg]);
            if (EXACT) {
              tma_load_2d(db + 2 * BB, &M.x, cb, jb, &full[stg]);
              tma_load_2d(db + 3 * BB, &M.x, cbo, jb, &full[stg]);
            }
          }
        }
        __syncwarp();
      }
    } else {
      // ---- consumers: warp (wc, wr) owns columns x0 + 32 wc + lane, rows y0 + 4 wr + i
      const Stencil& st = A.st;
      const double L0 = st.left[0], L1 = st.left[1], L2 = st.left[2], D = st.diag;
      const double R0 = st.right[0], R1 = st.right[1], R2 = st.right[2];
      const bool hr0 = st.has_right[0], hr1 = st.has_right[1], hr2 = st.has_right[2];
      double* __restrict__ uo = UPD ? (cur ? A.uo0 : A.uo1) : nullptr;
      double* __restrict__ ro = UPD ? (cur ? A.ro0 : A.ro1) : (cur ? A.ro1 : A.ro0);
      const int warp = tid >> 5, lane = tid & 31;
      const int wc = warp % kS3CG, wr = warp / kS3CG;
      // own column and (lanes 0 / 31) the neighbour column, as box indices from x0 - 1; lanes past
      // the tile read a clamped column (their values are never used)
      const int cme = 32 * wc + lane + 1;
      const int cld = min(cme, TXB - 2);
      const int cedge = min(lane == 0 ? 32 * wc : (lane == 31 ? 32 * wc + 33 : cme), TXB - 2);
      PlaneSeq seq;
      seq.start(w0, w1, Nz);
      double vm[kS3R], vc[kS3R + 2], vce[kS3R];  // planes z - 1 and z (with the y-halo rows), z edge column
      int x0 = 0, y0 = 0, tw = 0, th = 0, x = 0;
      bool colok = false;
      for (long long L = 0; seq.valid; ++L, seq.advance()) {
        const int q = seq.q;
        if (q == seq.zb - 1) {  // new segment
          x0 = (seq.tile % G.ntx) * TX;
          y0 = (seq.tile / G.ntx) * kS3TY;
          tw = min(TX, Nx - x0);
          th = min(kS3TY, Ny - y0);
          x = x0 + cme - 1;
          colok = cme - 1 < tw;
#pragma unroll
          for (int i = 0; i < kS3R; ++i) vm[i] = vce[i] = 0.0;
#pragma unroll
          for (int i = 0; i < kS3R + 2; ++i) vc[i] = 0.0;
        }
        const int stg = static_cast<int>(L % NS);
        mbar_wait(&full[stg], static_cast<unsigned>((L / NS) & 1));
        const double* su = smem + static_cast<size_t>(stg) * SST;
        // v of plane q: own column rows -1 .. 4 of the group (box rows 4 wr .. 4 wr + 5), and the
        // neighbour column rows 0 .. 3
        double vp[kS3R + 2], vpe[kS3R];
        const bool vq = q >= 0 && q < Nz;
        if (vq) {
          const long long r0 = static_cast<long long>(y0 - 1) + static_cast<long long>(q) * Ny;
          const int p0 = static_cast<int>(r0 & 1);  // parity of box row 0
          const int she = (x0 - 1) & 1, sho = (Nx + x0 - 1) & 1;
#pragma unroll
          for (int i = 0; i < kS3R + 2; ++i) {
            const int r = kS3R * wr + i;  // box row (y = y0 - 1 + r)
            const int par = (p0 ^ r) & 1;
            const int base = par * BUE + ((r + p0) >> 1) * TXB + (par ? sho : she);
            const double uv = su[base + cld];
            vp[i] = UPD ? __dadd_rn(uv, __dmul_rn(s, su[2 * BUE + base + cld])) : uv;
            if (i >= 1 && i <= kS3R) {
              const double ue = su[base + cedge];
              vpe[i - 1] = UPD ? __dadd_rn(ue, __dmul_rn(s, su[2 * BUE + base + cedge])) : ue;
            }
          }
        } else {
#pragma unroll
          for (int i = 0; i < kS3R + 2; ++i) vp[i] = 0.0;
#pragma unroll
          for (int i = 0; i < kS3R; ++i) vpe[i] = 0.0;
        }
        // residual of plane z = q - 1: v(z-1) = vm, v(z) = vc (+ halo rows, x neighbours by
        // shuffle / the edge column), v(z+1) = vp; b (and exact) of plane z from this stage
        const int z = q - 1;
        const bool outz = z >= seq.zb && colok;
        const bool zl = z > 0, zr = z < Nz - 1 && hr2;
        const double* sb = su + NUE * BUE;
        const long long rb0 = static_cast<long long>(y0) + static_cast<long long>(z) * Ny;
        const int pb = static_cast<int>(rb0 & 1);
        const int sbe = x0 & 1, sbo = (Nx + x0) & 1;
        const i64 gz = static_cast<i64>(z) * sxy + x + static_cast<i64>(y0 + kS3R * wr) * Nx;
#pragma unroll
        for (int i = 0; i < kS3R; ++i) {
          // (every lane takes part in both shuffles; lanes 0 / 31 then use the edge column)
          const double su_l = __shfl_up_sync(0xffffffffu, vc[i + 1], 1);
          const double su_r = __shfl_down_sync(0xffffffffu, vc[i + 1], 1);
          const double vl = lane == 0 ? vce[i] : su_l;
          const double vr = lane == 31 ? vce[i] : su_r;
          const int yr = kS3R * wr + i;  // tile row
          if (outz && yr < th) {
            const int y = y0 + yr;
            double acc = 0.0;
            if (zl) acc = __dadd_rn(acc, __dmul_rn(L2, vm[i]));
            if (y > 0) acc = __dadd_rn(acc, __dmul_rn(L1, vc[i]));
            if (x > 0) acc = __dadd_rn(acc, __dmul_rn(L0, vl));
            acc = __dadd_rn(acc, __dmul_rn(D, vc[i + 1]));
            if (x < Nx - 1 && hr0) acc = __dadd_rn(acc, __dmul_rn(R0, vr));
            if (y < Ny - 1 && hr1) acc = __dadd_rn(acc, __dmul_rn(R1, vc[i + 2]));
            if (zr) acc = __dadd_rn(acc, __dmul_rn(R2, vp[i + 1]));
            const int par = (pb ^ yr) & 1;
            const int ob = par * BB + ((yr + pb) >> 1) * TXB + (par ? sbo : sbe) + cme - 1;
            double r = __dsub_rn(sb[ob], acc);
            if (UPD && A.sparse && (x + 1) % A.n[0] != 0 && (y + 1) % A.n[1] != 0 && (z + 1) % A.n[2] != 0) r = 0.0;
            const i64 gp = gz + static_cast<i64>(i) * Nx;
            ro[gp] = r;
            if (UPD) uo[gp] = vc[i + 1];
            a0 += r * r;
            a1 = fmax(a1, fabs(r));
            if (EXACT) {
              const double d = vc[i + 1] - sb[2 * BB + ob];
              a2 += d * d;
              a3 = fmax(a3, fabs(d));
            }
          }
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(&empty[stg]);  // this warp is past its reads of the stage
#pragma unroll
        for (int i = 0; i < kS3R; ++i) {
          vm[i] = vc[i + 1];
          vce[i] = vpe[i];
        }
#pragma unroll
        for (int i = 0; i < kS3R + 2; ++i) vc[i] = vp[i];
      }
    }
  }
  block_reduce4_march(a0, a1, a2, a3, A.partials);
  fold_ctrl(A.ctrl, A.partials, S, A.history);
}

S3Geo s3_geo(const FineGeom& g) {
  S3Geo G{};
  G.ntx = (g.ext[0] + kS3MaxTX - 1) / kS3MaxTX;
  G.tx = (g.ext[0] + G.ntx - 1) / G.ntx;
  G.nty = (g.ext[1] + kS3TY - 1) / kS3TY;
  G.txb = (G.tx + 3 + 1) & ~1;  // TX + 2 halo columns + the alignment shift, even
  G.box_ue = ((kS3PairsUE * G.txb * 8 + 127) / 128) * 128 / 8;
  G.box_b = ((kS3PairsB * G.txb * 8 + 127) / 128) * 128 / 8;
  G.work = static_cast<long long>(G.ntx) * G.nty * g.ext[2];
  return G;
}

size_t s3_stage_doubles(const S3Geo& G, bool upd, bool exact) {
  return static_cast<size_t>(upd ? 4 : 2) * G.box_ue + static_cast<size_t>(exact ? 4 : 2) * G.box_b;
}

constexpr size_t kS3SmemMax = 227 * 1024 - 2304;  // beside the static shared memory of the reductions

using EncodeTiled = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                 const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                 CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeTiled encode_fn() {
  static EncodeTiled fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q{};
    ASDSM_CUDA_CHECK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess) throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeTiled>(p);
  }
  return fn;
}

// Pair-row view of a fine array: (2 N_x, ceil(N_y N_z / 2)) doubles, row stride 16 N_x bytes,
// boxes of `pairs` row pairs.  (The last pair's odd row lies past the array when N_y N_z is odd:
// fine arrays carry a row of slack, Solver::init.)
CUtensorMap pair_map(const double* base, const FineGeom& g, const S3Geo& G, int pairs) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * g.ext[0]),
                              static_cast<cuuint64_t>((static_cast<long long>(g.ext[1]) * g.ext[2] + 1) / 2)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * g.ext[0]) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(G.txb), static_cast<cuuint32_t>(pairs)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

template <bool UPD, bool EXACT>
void launch_variant(const MarchArgs& A, const S3Geo& G, const S3Maps& M, size_t smem, cudaStream_t s) {
  static size_t attr = 0;  // dynamic shared memory opted in so far
  if (smem > attr) {
    ASDSM_CUDA_CHECK(cudaFuncSetAttribute(stream3d_kernel<UPD, EXACT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(smem)));
    attr = smem;
  }
  const unsigned grid = static_cast<unsigned>(std::min<long long>(kNumSms, G.work));
  stream3d_kernel<UPD, EXACT><<<grid, kS3Threads, smem, s>>>(A, G, M);
}

}  // namespace

// ASDSM_STREAM3D=1 (read at launch / capture) selects this pass; the default is the axpy +
// z-coarsened residual passes (march.cu), measured faster for the update: config 4 1.83 vs
// 1.43 ms per update (2.9 vs 3.7 TB/s of the algorithmic 40 B/point) -- the residual mode alone
// matches the default (0.81 vs 0.83 ms, 3.9 TB/s).  See DESIGN.md "Measured and not kept".
bool stream3d_supported(const MarchArgs& A) {
  if (A.g.dim != 3 || A.coef != nullptr || A.g.stride[1] != A.g.ext[0] || !std::getenv("ASDSM_STREAM3D")) return false;
  S3Geo G = s3_geo(A.g);
  return 128 + 2 * s3_stage_doubles(G, true, A.exact != nullptr) * sizeof(double) <= kS3SmemMax;
}

void launch_stream3d(int mode, const MarchArgs& A, cudaStream_t s) {
  S3Geo G = s3_geo(A.g);
  const bool upd = mode == kMarchUpdate, exact = A.exact != nullptr;
  const size_t st = s3_stage_doubles(G, upd, exact) * sizeof(double);
  G.ns = kS3MaxStages;
  while (G.ns > 2 && 128 + G.ns * st > kS3SmemMax) --G.ns;
  const size_t smem = 128 + G.ns * st;
  if (smem > kS3SmemMax) throw AsdsmError(kUnsupported, "3D TMA pass: tile stages exceed shared memory");
  S3Maps M;
  M.u0 = pair_map(A.u0, A.g, G, kS3PairsUE);
  M.u1 = pair_map(A.u1, A.g, G, kS3PairsUE);
  M.e = upd ? pair_map(A.e, A.g, G, kS3PairsUE) : M.u0;
  M.b = pair_map(A.b, A.g, G, kS3PairsB);
  M.x = exact ? pair_map(A.exact, A.g, G, kS3PairsB) : M.b;
  if (upd && exact) launch_variant<true, true>(A, G, M, smem, s);
  else if (upd) launch_variant<true, false>(A, G, M, smem, s);
  else if (exact) launch_variant<false, true>(A, G, M, smem, s);
  else launch_variant<false, false>(A, G, M, smem, s);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
