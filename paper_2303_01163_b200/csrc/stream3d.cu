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
// stride is 16 N_x bytes: a tile's 18 rows (16 + the y halo) of one plane are two 2D boxes of
// 10 row pairs, the even rows at x offset x0 - 1 and the odd rows at N_x + x0 - 1 (out-of-range
// boxes are zero-filled by the TMA unit; the values it reads across a row end are never used).
// A producer warp issues 4 TMA loads per plane (u, e x even, odd) on a 4-stage mbarrier ring,
// 3 planes in flight; 16 consumer warps form v = u + s e once per point (halo included) into a
// 3-plane ring, so each v value costs one read of u and e: the pass moves u, e, b in and u', r
// out -- 40 B per point (+8 with an exact solution) plus the re-read y-halo rows.  The row sum
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

constexpr int kS3Cons = 512;                 // consumer threads
constexpr int kS3Threads = kS3Cons + 32;     // + one producer warp
constexpr int kS3TY = 16;                    // tile rows
constexpr int kS3Rows = kS3TY + 2;           // with the y halo
constexpr int kS3Pairs = 10;                 // row pairs per box (covers 18 rows at any parity)
constexpr int kS3MaxStages = 4;              // TMA pipeline depth (planes), at most
constexpr int kS3MaxTX = 128;
constexpr int kS3RG = kS3Cons / kS3MaxTX;    // row groups (4)
constexpr int kS3Pts = kS3TY / kS3RG;        // points per consumer thread (4)

struct S3Geo {
  int tx, ntx, nty;  // tile width, tiles along x / y
  int txb;           // box width (doubles): TX + 3 rounded up to even
  int box;           // doubles per box in shared memory (128-byte aligned)
  int vw;            // v-ring row stride: TX + 2
  long long work;    // ntx * nty * Nz planes
  int ns;            // pipeline stages that fit beside the v ring and the b slots (2..4)
  int probe;         // ASDSM_S3_PROBE (measurement only): 1 = loads without compute, 2 = compute without
                     // loads, 3 = no stores (interior), 4 = no b loads
};

struct S3Maps {  // tensor maps of the pair-row views (u0, u1, e)
  CUtensorMap u0, u1, e;
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
__device__ __forceinline__ void consumer_sync() { asm volatile("bar.sync 1, %0;" ::"n"(kS3Cons) : "memory"); }

// The sequence of planes one CTA loads: its share [w0, w1) of the flattened (tile, z) space
// as per-tile segments [zb, ze); a segment loads planes zb-1 .. ze (virtual -- no copy --
// outside [0, Nz)).  Producer and consumers walk identical copies.
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

template <bool UPD>
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
  const Stencil& st = A.st;
  double* __restrict__ uo = UPD ? (cur ? A.uo0 : A.uo1) : nullptr;
  double* __restrict__ ro = UPD ? (cur ? A.ro0 : A.ro1) : (cur ? A.ro1 : A.ro0);
  const int TX = G.tx, VW = G.vw, BOX = G.box, TXB = G.txb;
  constexpr int NARR = UPD ? 2 : 1;
  const int SBOX = 2 * NARR * BOX;  // doubles per stage

  extern __shared__ __align__(128) double smem_raw[];
  // TMA destinations 128-byte aligned (the dynamic window follows the static shared variables)
  // (an integer offset from the shared array, not an integer-cast pointer: the compiler keeps
  // every access in the shared state space -- LDS/STS with 32-bit addressing)
  double* smem = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u) / sizeof(double);
  double* stage = smem;                                                // [NS][array][parity][pair][TXB]
  const int NS = G.ns;
  double* vring = smem + static_cast<size_t>(NS) * SBOX;              // [3][18][VW]
  // b (and exact) of the thread's own points, one plane ahead: [slot][array][k][consumer]
  double* bsl = vring + 3 * kS3Rows * VW;
  __shared__ __align__(8) unsigned long long full[kS3MaxStages], empty[kS3MaxStages];

  const int tid = threadIdx.x;
  const long long w0 = G.work * blockIdx.x / gridDim.x, w1 = G.work * (blockIdx.x + 1) / gridDim.x;
  if (tid == 0) {
    for (int i = 0; i < NS; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  if (work && w0 < w1) {
    if (tid >= kS3Cons) {
      // ---- producer warp: plane load L into stage L % NS once the consumers released it.  The
      // whole warp walks the loop (lane 0 issues): a lone lane whose siblings already sit at the
      // final CTA barrier is scheduled only sporadically, which stalled every plane hand-off
      {
        const bool leader = tid == kS3Cons;
        PlaneSeq prod;
        prod.start(w0, w1, Nz);
        long long L = 0;
        for (; prod.valid; prod.advance()) {
          const int q = prod.q;
          if (q < 0 || q >= Nz) continue;  // virtual plane: no load
          const int stg = static_cast<int>(L % NS);
          if (L >= NS) mbar_wait(&empty[stg], static_cast<unsigned>(((L / NS) - 1) & 1));
          const int x0 = (prod.tile % G.ntx) * TX, y0 = (prod.tile / G.ntx) * kS3TY;
          const long long r0 = static_cast<long long>(y0 - 1) + static_cast<long long>(q) * Ny;  // first row
          const int j0 = static_cast<int>(r0 >= 0 ? r0 >> 1 : -1);
          if (leader && G.probe == 2) mbar_arrive(&full[stg]);
          if (leader && G.probe != 2) {
          mbar_arrive_expect_tx(&full[stg], static_cast<unsigned>(2 * NARR * kS3Pairs * TXB * 8));
          double* d = stage + static_cast<size_t>(stg) * SBOX;
          // box x origins 16-byte aligned (the TMA unit requires it): the even coordinate at or
          // before x0 - 1 (even rows) and N_x + x0 - 1 (odd rows); consumers add the shift back
          const int ce = (x0 - 1) & ~1, co = (Nx + x0 - 1) & ~1;
          // (the buffer is picked by a branch, not a pointer select: the tensor map operand must
          // stay a kernel-parameter address, never a local copy)
          if (cur) {
            tma_load_2d(d, &M.u1, ce, j0, &full[stg]);
            tma_load_2d(d + BOX, &M.u1, co, j0, &full[stg]);
          } else {
            tma_load_2d(d, &M.u0, ce, j0, &full[stg]);
            tma_load_2d(d + BOX, &M.u0, co, j0, &full[stg]);
          }
          if (UPD) {
            tma_load_2d(d + 2 * BOX, &M.e, ce, j0, &full[stg]);
            tma_load_2d(d + 3 * BOX, &M.e, co, j0, &full[stg]);
          }
          }
          ++L;
          __syncwarp();
        }
      }
    } else {
      // ---- consumers: thread (cx, rg) owns column x0 + cx, rows rg + 4k of the tile
      const int cx = tid & (kS3MaxTX - 1), rg = tid / kS3MaxTX;
      const double L0 = st.left[0], L1 = st.left[1], L2 = st.left[2], D = st.diag;
      const double R0 = st.right[0], R1 = st.right[1], R2 = st.right[2];
      PlaneSeq seq;
      seq.start(w0, w1, Nz);
      long long L = 0;
      int vslot = 0;  // ring slot of plane q
      double vm[kS3Pts], vc[kS3Pts];
      int x0 = 0, y0 = 0, th = 0, hw = 0, cofs = 0, she = 0, sho = 0;
      unsigned ownm = 0, rowm = 0;  // own points k; halo rows r = rg + 4i inside the grid
      bool colok = false, fast = false, extra = false;
      const int vown = (rg + 1) * VW + cx + 1;  // ring index of own point k = 0
      double* const bown = bsl + tid;
      while (seq.valid) {
        const int q = seq.q;
        if (q == seq.zb - 1) {  // new segment: tile geometry, masks, registers cleared
          x0 = (seq.tile % G.ntx) * TX;
          y0 = (seq.tile / G.ntx) * kS3TY;
          const int tw = min(TX, Nx - x0);
          th = min(kS3TY, Ny - y0);
          hw = min(tw + 2, Nx - x0 + 1);  // halo columns c = x - (x0 - 1) inside the grid
          extra = cx + kS3MaxTX < hw;
          cofs = x0 + cx + (y0 + rg) * Nx;  // in-plane offset of point k = 0
          colok = cx < tw;
          she = (x0 - 1) & 1;
          sho = (Nx + x0 - 1) & 1;  // TMA box origin shifts (see the producer)
          ownm = 0;
#pragma unroll
          for (int k = 0; k < kS3Pts; ++k)
            if (colok && rg + kS3RG * k < th) ownm |= 1u << k;
          rowm = 0;
          for (int i = 0; rg + kS3RG * i < kS3Rows; ++i) {
            const int y = y0 - 1 + rg + kS3RG * i;
            if (y >= 0 && y < Ny && cx < hw) rowm |= 1u << i;
          }
          const int x = x0 + cx;
          // interior points: every x / y stencil term present for all four points
          fast = ownm == (1u << kS3Pts) - 1 && x > 0 && x < Nx - 1 && st.has_right[0] && y0 + rg > 0 &&
                 y0 + rg + kS3RG * (kS3Pts - 1) < Ny - 1 && st.has_right[1] && !(UPD && A.sparse);
#pragma unroll
          for (int k = 0; k < kS3Pts; ++k) vm[k] = vc[k] = 0.0;
        }
        const int stg = static_cast<int>(L % NS);
        const bool vq = q >= 0 && q < Nz;
        // b (and exact) of plane q: cp.async into this thread's slot (q & 1) now, read back next
        // step (the residual of plane q) after the group completed -- no register waits on them
        if (q >= seq.zb && q < seq.ze && ownm && G.probe != 4) {
          const i64 gq = static_cast<i64>(q) * sxy + cofs;
          double* bs = bown + (q & 1) * (2 * kS3Pts * kS3Cons);
#pragma unroll
          for (int k = 0; k < kS3Pts; ++k) {
            if (ownm & (1u << k)) {
              cp_async8(bs + k * kS3Cons, A.b + gq + kS3RG * k * Nx);
              if (A.exact) cp_async8(bs + (kS3Pts + k) * kS3Cons, A.exact + gq + kS3RG * k * Nx);
            }
          }
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
        // v of plane q over the halo tile into ring slot vslot
        double* V = vring + vslot * (kS3Rows * VW);
        if (vq) {
          mbar_wait(&full[stg], static_cast<unsigned>((L / NS) & 1));
          if (G.probe != 1) {
            const double* su = stage + stg * SBOX;
            const int p0 = static_cast<int>((y0 - 1 + static_cast<long long>(q) * Ny) & 1);  // first row's parity
#pragma unroll
            for (int i = 0; i < (kS3Rows + kS3RG - 1) / kS3RG; ++i) {
              if (!(rowm & (1u << i))) continue;
              const int r = rg + kS3RG * i;
              const int par = (p0 ^ r) & 1;
              const int off = par * BOX + ((r + p0) >> 1) * TXB + (par ? sho : she) + cx;
              const double uv = su[off];
              V[r * VW + cx] = UPD ? __dadd_rn(uv, __dmul_rn(s, su[2 * BOX + off])) : uv;
              if (extra) {
                const double uw = su[off + kS3MaxTX];
                V[r * VW + cx + kS3MaxTX] = UPD ? __dadd_rn(uw, __dmul_rn(s, su[2 * BOX + off + kS3MaxTX])) : uw;
              }
            }
          }
        }
        consumer_sync();
        if (vq && tid == 0) mbar_arrive(&empty[stg]);  // every consumer is past its reads
        if (G.probe == 1) {
          vslot = vslot == 2 ? 0 : vslot + 1;
          if (vq) ++L;
          seq.advance();
          continue;
        }
        // residual of plane z = q - 1 with v(z-1) = vm, v(z) = vc, v(z+1) = V (ring slot vslot)
        const int z = q - 1;
        const double* Vz = vring + (vslot == 0 ? 2 : vslot - 1) * (kS3Rows * VW) + vown;
        const double* Vq = V + vown;
        asm volatile("cp.async.wait_group 1;" ::: "memory");  // plane z's b group is complete
        const double* bz = bown + (z & 1) * (2 * kS3Pts * kS3Cons);
        const bool outz = z >= seq.zb;
        const bool zl = z > 0, zr = z < Nz - 1 && st.has_right[2];
        const i64 gz = static_cast<i64>(z) * sxy + cofs;
        if (fast && vq && outz) {
          // interior column: straight-line stencil rows (the reference's CSR order, fdm.cpp:110-117)
#pragma unroll
          for (int k = 0; k < kS3Pts; ++k) {
            const double* c = Vz + k * (kS3RG * VW);
            const double vp = Vq[k * (kS3RG * VW)];
            double acc = __dadd_rn(0.0, __dmul_rn(L2, zl ? vm[k] : 0.0));
            if (!zl) acc = 0.0;
            acc = __dadd_rn(acc, __dmul_rn(L1, c[-VW]));
            acc = __dadd_rn(acc, __dmul_rn(L0, c[-1]));
            acc = __dadd_rn(acc, __dmul_rn(D, vc[k]));
            acc = __dadd_rn(acc, __dmul_rn(R0, c[1]));
            acc = __dadd_rn(acc, __dmul_rn(R1, c[VW]));
            if (zr) acc = __dadd_rn(acc, __dmul_rn(R2, vp));
            const double r = __dsub_rn(bz[k * kS3Cons], acc);
            const i64 gp = gz + kS3RG * k * Nx;
            if (G.probe != 3) {
              ro[gp] = r;
              if (UPD) uo[gp] = vc[k];
            }
            a0 += r * r;
            a1 = fmax(a1, fabs(r));
            if (A.exact) {
              const double d = vc[k] - bz[(kS3Pts + k) * kS3Cons];
              a2 += d * d;
              a3 = fmax(a3, fabs(d));
            }
            vm[k] = vc[k];
            vc[k] = vp;
          }
        } else {
#pragma unroll
          for (int k = 0; k < kS3Pts; ++k) {
            const bool own = ownm & (1u << k);
            const double vp = (own && vq) ? Vq[k * (kS3RG * VW)] : 0.0;
            if (outz && own) {
              const int x = x0 + cx, y = y0 + rg + kS3RG * k;
              const double* c = Vz + k * (kS3RG * VW);
              double acc = 0.0;
              if (zl) acc = __dadd_rn(acc, __dmul_rn(L2, vm[k]));
              if (y > 0) acc = __dadd_rn(acc, __dmul_rn(L1, c[-VW]));
              if (x > 0) acc = __dadd_rn(acc, __dmul_rn(L0, c[-1]));
              acc = __dadd_rn(acc, __dmul_rn(D, vc[k]));
              if (x < Nx - 1 && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(R0, c[1]));
              if (y < Ny - 1 && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(R1, c[VW]));
              if (zr) acc = __dadd_rn(acc, __dmul_rn(R2, vp));
              double r = __dsub_rn(bz[k * kS3Cons], acc);
              if (UPD && A.sparse && (x + 1) % A.n[0] != 0 && (y + 1) % A.n[1] != 0 && (z + 1) % A.n[2] != 0) r = 0.0;
              const i64 gp = gz + kS3RG * k * Nx;
              ro[gp] = r;
              if (UPD) uo[gp] = vc[k];
              a0 += r * r;
              a1 = fmax(a1, fabs(r));
              if (A.exact) {
                const double d = vc[k] - bz[(kS3Pts + k) * kS3Cons];
                a2 += d * d;
                a3 = fmax(a3, fabs(d));
              }
            }
            vm[k] = vc[k];
            vc[k] = vp;
          }
        }
        vslot = vslot == 2 ? 0 : vslot + 1;
        if (vq) ++L;
        seq.advance();
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
  G.box = ((kS3Pairs * G.txb * 8 + 127) / 128) * 128 / 8;
  G.vw = G.tx + 2;
  G.work = static_cast<long long>(G.ntx) * G.nty * g.ext[2];
  G.probe = std::getenv("ASDSM_S3_PROBE") ? std::atoi(std::getenv("ASDSM_S3_PROBE")) : 0;
  return G;
}

size_t s3_smem(const S3Geo& G, bool upd, int ns) {
  return 128 + sizeof(double) * (static_cast<size_t>(ns) * 2 * (upd ? 2 : 1) * G.box + 3u * kS3Rows * G.vw +
                                 2u * 2 * kS3Pts * kS3Cons);
}

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

// Pair-row view of a fine array: (2 N_x, ceil(N_y N_z / 2)) doubles, row stride 16 N_x bytes.
// (The last pair's odd row lies past the array when N_y N_z is odd: fine arrays carry a row of
// slack, Solver::alloc_fine.)
CUtensorMap pair_map(const double* base, const FineGeom& g, const S3Geo& G) {
  CUtensorMap m;
  std::memset(&m, 0, sizeof(m));
  const cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * g.ext[0]),
                              static_cast<cuuint64_t>((static_cast<long long>(g.ext[1]) * g.ext[2] + 1) / 2)};
  const cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * g.ext[0]) * sizeof(double)};
  const cuuint32_t box[2] = {static_cast<cuuint32_t>(G.txb), static_cast<cuuint32_t>(kS3Pairs)};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode_fn()(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double*>(base), dims, strides, box,
                                 estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

}  // namespace

// Opt-in (ASDSM_STREAM3D=1, read at launch / capture): measured slower than the default axpy +
// z-coarsened residual passes (config 4 update 1.57 vs 1.43 ms, config 3 0.34 vs 0.26 ms; see
// DESIGN.md "Measured and not kept") -- the per-plane consumer barrier and ~150 issued
// instructions per point keep 17 warps per SM at ~2.2 IPC, so the kernel is issue-bound well
// before HBM; kept with its parity tests as the TMA pair-row staging reference.
bool stream3d_supported(const MarchArgs& A) {
  return A.g.dim == 3 && A.coef == nullptr && A.g.stride[1] == A.g.ext[0] && std::getenv("ASDSM_STREAM3D") != nullptr;
}

void launch_stream3d(int mode, const MarchArgs& A, cudaStream_t s) {
  const S3Geo G = s3_geo(A.g);
  const bool upd = mode == kMarchUpdate;
  S3Geo G2 = G;
  G2.ns = kS3MaxStages;
  while (G2.ns > 2 && s3_smem(G2, upd, G2.ns) + 2304 > 227u * 1024) --G2.ns;
  const size_t smem = s3_smem(G2, upd, G2.ns);
  static size_t attr_set[2] = {0, 0};  // dynamic shared memory opted in so far, per variant
  if (smem > attr_set[upd]) {
    if (upd) ASDSM_CUDA_CHECK(cudaFuncSetAttribute(stream3d_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    else ASDSM_CUDA_CHECK(cudaFuncSetAttribute(stream3d_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
    attr_set[upd] = smem;
  }
  S3Maps M;
  M.u0 = pair_map(A.u0, A.g, G);
  M.u1 = pair_map(A.u1, A.g, G);
  M.e = upd ? pair_map(A.e, A.g, G) : M.u0;
  const unsigned grid = static_cast<unsigned>(std::min<long long>(kNumSms, G.work));
  if (upd) stream3d_kernel<true><<<grid, kS3Threads, smem, s>>>(A, G2, M);
  else stream3d_kernel<false><<<grid, kS3Threads, smem, s>>>(A, G2, M);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
