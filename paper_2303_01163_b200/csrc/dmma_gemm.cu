// DMMA (fp64 tensor-pipe mma.sync) transform GEMM for sm_100a.  Same FP64 peak as DFMA on
// B200 (both ~37 TFLOP/s measured), but each 8x8x4 MMA takes one A and one B operand
// per lane, so a 32x32 warp tile needs 8 shared-memory loads per 16 MMAs (4096 FMAs) --
// the scalar register-tiled kernel is limited by shared-memory bandwidth instead.
#include "dmma_gemm.cuh"

#include <algorithm>
#include <cstdlib>

namespace asdsm_b200 {

namespace {

constexpr int BP = 64, BQ = 64, BK = 32, PAD = 4, NTH = 128;

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void line_base(const GemmLines& L, i64 p, i64& ib, i64& ob) {
  i64 o0, o1, h0, h1, h2;
  if (L.nlines < (i64{1} << 31)) {  // 32-bit divisions: five 64-bit ones open every tile otherwise
    const unsigned e0 = static_cast<unsigned>(L.o_ext[0]), e1 = static_cast<unsigned>(L.o_ext[1]);
    const unsigned b0 = static_cast<unsigned>(L.nbox[0]), b1 = static_cast<unsigned>(L.nbox[1]);
    unsigned t = static_cast<unsigned>(p), q = t / e0;
    o0 = t - q * e0;
    t = q;
    q = t / e1;
    o1 = t - q * e1;
    t = q;
    q = t / b0;
    h0 = t - q * b0;
    t = q;
    q = t / b1;
    h1 = t - q * b1;
    h2 = q;
  } else {
    o0 = p % L.o_ext[0];
    i64 t = p / L.o_ext[0];
    o1 = t % L.o_ext[1];
    t /= L.o_ext[1];
    h0 = t % L.nbox[0];
    t /= L.nbox[0];
    h1 = t % L.nbox[1];
    h2 = t / L.nbox[1];
  }
  ib = h0 * L.in_bs[0] + h1 * L.in_bs[1] + h2 * L.in_bs[2] + o0 * L.o_in[0] + o1 * L.o_in[1];
  ob = h0 * L.out_bs[0] + h1 * L.out_bs[1] + h2 * L.out_bs[2] + o0 * L.o_out[0] + o1 * L.o_out[1];
}

#ifndef ASDSM_DENSE_MINB
#define ASDSM_DENSE_MINB 3  // 168 registers, three CTAs per SM (config 4: 54.0 -> 53.8 ms)
#endif
template <bool kContigIn, bool kContigOut>
__global__ void __launch_bounds__(NTH, ASDSM_DENSE_MINB) dmma_transform_kernel(const double* __restrict__ in, double* __restrict__ out,
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
    auto kstep = [&](int kk) {
      double a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[wp + i * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[wq + j * 8 + (lane >> 2)][kk + (lane & 3)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    };
    if (k0 + BK <= m) {
#pragma unroll
      for (int kk = 0; kk < BK; kk += 4) kstep(kk);
    } else {  // last tile: only the k groups that hold modes (the rest of the tile is zeros)
      for (int kk = 0; k0 + kk < m; kk += 4) kstep(kk);
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


// Even/odd-split transforms (plan.cpp half_sine_tables): V = D S and W = c S D^-1 with S the
// DST-I matrix, whose row m-1-i is (-1)^k times row i.  Both directions need only the
// ceil(m/2) x m half table SH (even columns first, then odd) and half the MMAs of the dense
// GEMM:
//   back:    E_q = sum_kappa x_{2 kappa} SH[q][kappa],  O_q = sum_kappa x_{2 kappa+1} SH[q][kh+kappa]
//            out(q) = sc_q (E_q + O_q),  out(m-1-q) = sc_{m-1-q} (E_q - O_q)      (q < ceil(m/2))
//   forward: g_j = ci_j in(j),  h+-_j = g_j +- g_{m-1-j}  (j < ceil(m/2); h = g_j at j = m-1-j)
//            out(2 kappa) = sum_j h+_j SH[j][kappa],  out(2 kappa+1) = sum_j h-_j SH[j][kh+kappa]
// Warp-specialized: warps 0-3 accumulate E, warps 4-7 O over the same 64 x 64 tile (each warp
// 32 x 32, the dense kernel's register budget); the back transform combines them through shared
// memory in the epilogue.
constexpr int EP = 64, EQ = 64, EK = 16, ELD2 = EK + 4, ENT2 = 256;
constexpr size_t kEo2Smem = sizeof(double) * 4 * EP * ELD2 + 2 * EP * sizeof(i64);

template <bool kBack, bool kContigIn, int EQT>
__global__ void __launch_bounds__(ENT2, 2) dmma_eo2_kernel(const double* __restrict__ in, double* __restrict__ out,
                                                           const double* __restrict__ SH, const double* __restrict__ sc,
                                                           int m, int kh, i64 in_es, i64 out_es, GemmLines L) {
  extern __shared__ __align__(16) double esm[];
  double(*AE)[ELD2] = reinterpret_cast<double(*)[ELD2]>(esm);
  double(*AO)[ELD2] = reinterpret_cast<double(*)[ELD2]>(esm + EP * ELD2);
  double(*BE)[ELD2] = reinterpret_cast<double(*)[ELD2]>(esm + 2 * EP * ELD2);
  double(*BO)[ELD2] = reinterpret_cast<double(*)[ELD2]>(esm + 3 * EP * ELD2);
  i64* s_ib = reinterpret_cast<i64*>(esm + 4 * EP * ELD2);
  i64* s_ob = s_ib + EP;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int grp = warp >> 2, wl = warp & 3;  // grp 0: E, 1: O
  constexpr int NB = EQT / 16;  // 8-wide n tiles per warp (the warp tile is 32 x EQT / 2)
  const int wp = (wl >> 1) * 32, wq = (wl & 1) * (EQT / 2);
  const int mh = (m + 1) >> 1;
  const i64 p0 = static_cast<i64>(blockIdx.y) * EP;
  const int q0 = blockIdx.x * EQT;
  const double* __restrict__ ci = sc + m;
  for (int t = tid; t < EP; t += ENT2) {
    i64 ib = 0, ob = 0;
    if (p0 + t < L.nlines) line_base(L, p0 + t, ib, ob);
    s_ib[t] = ib;
    s_ob[t] = ob;
  }
  __syncthreads();
  double acc[4][NB][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < NB; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
  const int K = kBack ? kh : mh;
  constexpr int PA = (EP * 2 * EK) / ENT2;  // 8
  constexpr int PB = (EQT * 2 * EK) / ENT2;  // 8 (6)
  double ra[PA], rb[PB];
  auto load = [&](int k0) {
    if (kBack) {
#pragma unroll
      for (int r = 0; r < PA; ++r) {
        const int e = tid + r * ENT2;
        int pl, c;  // c in [0, 2 EK): mode 2 k0 + c
        if (kContigIn) {
          pl = e / (2 * EK);
          c = e % (2 * EK);
        } else {
          pl = e % EP;
          c = e / EP;
        }
        double v = 0.0;
        if (p0 + pl < L.nlines) {
          const int k = 2 * k0 + c;
          if (k < m) v = __ldg(in + s_ib[pl] + static_cast<i64>(k) * in_es);
        }
        ra[r] = v;
      }
    } else {
      // forward: a thread loads the pair g_j = ci_j in(j), g_{m-1-j} of its (line, j) elements, so
      // h+ / h- are formed in registers when the tile is stored (no combine pass over the tile)
#pragma unroll
      for (int r = 0; r < PA / 2; ++r) {
        const int e = tid + r * ENT2;
        int pl, jl;
        if (kContigIn) {
          pl = e / EK;
          jl = e % EK;
        } else {
          pl = e % EP;
          jl = e / EP;
        }
        const int j = k0 + jl, jm = m - 1 - j;
        // raw values only: the ci factors are applied in store(), so no arithmetic waits on
        // these loads before the MMA loop of the current tile (the product here stalled every
        // warp on its global loads: long_scoreboard 40 % of the forward kernel's samples)
        double g = 0.0, gm = 0.0;
        if (p0 + pl < L.nlines && j < mh) {
          g = __ldg(in + s_ib[pl] + static_cast<i64>(j) * in_es);
          gm = jm == j ? 0.0 : __ldg(in + s_ib[pl] + static_cast<i64>(jm) * in_es);
        }
        ra[2 * r] = g;
        ra[2 * r + 1] = gm;
      }
    }
#pragma unroll
    for (int r = 0; r < PB; ++r) {
      const int e = tid + r * ENT2;
      double v = 0.0;
      if (kBack) {  // B(n = q, k = kappa): SH[q][half kh + kappa], kappa contiguous
        const int ql = e / (2 * EK), c = e % (2 * EK), half = c / EK, kl = c % EK;
        if (q0 + ql < mh && k0 + kl < kh) v = __ldg(SH + static_cast<i64>(q0 + ql) * 2 * kh + half * kh + k0 + kl);
      } else {  // B(n = kappa, k = j): SH[j][half kh + kappa], kappa contiguous
        const int nl = e % EQT, c = e / EQT, half = c / EK, jl = c % EK;
        if (q0 + nl < kh && k0 + jl < mh) v = __ldg(SH + static_cast<i64>(k0 + jl) * 2 * kh + half * kh + q0 + nl);
      }
      rb[r] = v;
    }
  };
  auto store = [&](int k0s) {
    if (kBack) {
#pragma unroll
      for (int r = 0; r < PA; ++r) {
        const int e = tid + r * ENT2;
        int pl, c;
        if (kContigIn) {
          pl = e / (2 * EK);
          c = e % (2 * EK);
        } else {
          pl = e % EP;
          c = e / EP;
        }
        if (c & 1) AO[pl][c >> 1] = ra[r];
        else AE[pl][c >> 1] = ra[r];
      }
    } else {
#pragma unroll
      for (int r = 0; r < PA / 2; ++r) {
        const int e = tid + r * ENT2;
        int pl, jl;
        if (kContigIn) {
          pl = e / EK;
          jl = e % EK;
        } else {
          pl = e % EP;
          jl = e / EP;
        }
        // g_j = ci_j in(j); h+ = g_j + g_{m-1-j}, h- = g_j - g_{m-1-j}; the middle row alone (its
        // mirror loaded as 0: g + 0 and g - 0 are g); beyond the half (raw values 0) both are 0
        const int j = k0s + jl;
        const double cj = j < mh ? __ldg(ci + j) : 0.0, cm = j < mh ? __ldg(ci + (m - 1 - j)) : 0.0;
        const double g = ra[2 * r] * cj, gm = ra[2 * r + 1] * cm;
        AE[pl][jl] = g + gm;
        AO[pl][jl] = g - gm;
      }
    }
#pragma unroll
    for (int r = 0; r < PB; ++r) {
      const int e = tid + r * ENT2;
      if (kBack) {
        const int ql = e / (2 * EK), c = e % (2 * EK);
        if (c < EK) BE[ql][c] = rb[r];
        else BO[ql][c - EK] = rb[r];
      } else {
        const int nl = e % EQT, c = e / EQT;
        if (c < EK) BE[nl][c] = rb[r];
        else BO[nl][c - EK] = rb[r];
      }
    }
  };
  const int r8 = lane >> 2, c4 = lane & 3;
  double(*As)[ELD2] = grp ? AO : AE;
  double(*Bs)[ELD2] = grp ? BO : BE;
  load(0);
  for (int k0 = 0; k0 < K; k0 += EK) {
    store(k0);
    __syncthreads();
    if (k0 + EK < K) load(k0 + EK);
    auto kstep = [&](int kk) {
      double fa[4], fb[NB];
#pragma unroll
      for (int a = 0; a < 4; ++a) fa[a] = As[wp + a * 8 + r8][kk + c4];
#pragma unroll
      for (int b = 0; b < NB; ++b) fb[b] = Bs[wq + b * 8 + r8][kk + c4];
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) dmma(acc[a][b], fa[a], fb[b]);
    };
    if (k0 + EK <= K) {
#pragma unroll
      for (int kk = 0; kk < EK; kk += 4) kstep(kk);
    } else {  // last tile: only the k groups below K (the rest of the tile is zeros)
      for (int kk = 0; k0 + kk < K; kk += 4) kstep(kk);
    }
    __syncthreads();
  }
  if (kBack) {
    // E -> shared (over the A tiles), then the O warps combine: out(q), out(m-1-q)
    double(*Ex)[EQT + 4] = reinterpret_cast<double(*)[EQT + 4]>(esm);
    if (grp == 0) {
#pragma unroll
      for (int a = 0; a < 4; ++a)
#pragma unroll
        for (int b = 0; b < NB; ++b) {
          Ex[wp + a * 8 + r8][wq + b * 8 + 2 * c4] = acc[a][b][0];
          Ex[wp + a * 8 + r8][wq + b * 8 + 2 * c4 + 1] = acc[a][b][1];
        }
    }
    __syncthreads();
    if (grp == 1) {
#pragma unroll
      for (int a = 0; a < 4; ++a) {
        const int pl = wp + a * 8 + r8;
        if (p0 + pl >= L.nlines) continue;
        const i64 ob = s_ob[pl];
#pragma unroll
        for (int b = 0; b < NB; ++b)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int ql = wq + b * 8 + 2 * c4 + h, q = q0 + ql;
            if (q >= mh) continue;
            const double E = Ex[pl][ql], O = acc[a][b][h];
            out[ob + static_cast<i64>(q) * out_es] = __ldg(sc + q) * (E + O);
            const int qm = m - 1 - q;
            if (qm != q) out[ob + static_cast<i64>(qm) * out_es] = __ldg(sc + qm) * (E - O);
          }
      }
    }
  } else {
#pragma unroll
    for (int a = 0; a < 4; ++a) {
      const int pl = wp + a * 8 + r8;
      if (p0 + pl >= L.nlines) continue;
      const i64 ob = s_ob[pl];
#pragma unroll
      for (int b = 0; b < NB; ++b)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int kap = q0 + wq + b * 8 + 2 * c4 + h;
          const int k = 2 * kap + grp;  // E -> even modes, O -> odd
          if (kap < kh && k < m) out[ob + static_cast<i64>(k) * out_es] = acc[a][b][h];
        }
    }
  }
}


// Back transform of a batch of hole strips with the half sine table resident in shared memory
// (config 2: 500 strips of w = 81 columns x 409 rows per iteration).  The generic even/odd kernel
// above re-stages the table for every 64 x 64 x 16 step and pads the 41 outputs of a strip's
// half transform to a 64-wide tile; here a CTA takes one (strip, row tile) work item:
//   modes [strip][k][j] (j contiguous) -> A tile [k in even/odd order][TR rows] by 8-byte cp.async
//   (the whole K extent at once: no K loop over global memory), the table once per CTA,
//   a warp pair 16 rows x every output (each warp half of the n tiles): E and O accumulators of the same (j, q) live in the same
//   thread, so out(q) = sc_q (E + O), out(m-1-q) = sc_{m-1-q} (E - O) needs no exchange and is
//   written straight from the accumulators.  One persistent CTA per SM walks the work items with
//   two A tiles in flight (the next tile's cp.async group is issued before this tile's MMAs).
//   The last row tile of a strip is shifted up to end at the strip's last row (it recomputes a
//   few rows of its neighbour -- the same values), so every tile is full.
struct StripBackArgs {
  int m, m1, kh, mh, ne, no4;  // modes, rows, padded half width, ceil(m/2), even modes, odd modes padded to 4
  int tiles;                   // row tiles per strip
  int nbox0, nboxes;
  i64 out_bs0, out_bs1, out_stride;
};

template <int NTW>  // n tiles of 8 outputs per warp: a warp pair covers 2 NTW >= ceil(mh / 8) tiles
__global__ void __launch_bounds__(512) strip_back_kernel(const double* __restrict__ modes, double* __restrict__ e,
                                                         const double* __restrict__ half, StripBackArgs P) {
  extern __shared__ __align__(16) double ssm[];
  const int tid = threadIdx.x, nth = blockDim.x, lane = tid & 31, warp = tid >> 5, nwarp = nth >> 5;
  const int TR = nth >> 2;  // 16 rows per warp pair
  const int LDA = TR + 4, LDB = 2 * P.kh + 4;
  const int m = P.m, m1 = P.m1, kh = P.kh, KA = kh + P.no4;
  double* Bs = ssm;                      // [16 NTW][LDB]: table row q, column half * kh + kappa
  double* Ss = Bs + 16 * NTW * LDB;      // sc[m]
  double* Ab = Ss + ((m + 1) & ~1);      // two A tiles [KA][LDA]: even modes, then odd modes
  const int ntile = P.tiles * P.nboxes;
  // the tile's modes, every k at once, by 8-byte cp.async: this warp's share is rows k = warp,
  // warp + nwarp, ... in chunks of 32 rows-of-j; item i = (row i / nch, chunk i % nch)
  // The issue state walks (k, chunk) incrementally -- a division and a modulo by nch per item were
  // 29 % of the kernel's instructions in the ncu source page -- and the shared address is formed
  // from a 32-bit base instead of a generic-to-shared conversion per copy.
  const int nch = (TR + 31) >> 5;
  int ik = warp, ic = 0;
  auto issue_item = [&](const double* __restrict__ src, unsigned as_s) {
    const int j = 32 * ic + lane;
    const int row = (ik & 1) ? kh + (ik >> 1) : (ik >> 1);
    if (j < TR)
      asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(as_s + 8u * static_cast<unsigned>(row * LDA + j)),
                   "l"(src + static_cast<i64>(ik) * m1 + j));
    if (++ic == nch) {
      ic = 0;
      ik += nwarp;
    }
  };
  auto tile_src = [&](int tile) {
    const int box = tile / P.tiles, t = tile - box * P.tiles;
    return modes + static_cast<i64>(box) * m * m1 + min(t * TR, m1 - TR);
  };
  const double* __restrict__ sc = half + static_cast<i64>(half_sine_rows(m)) * 2 * kh;
  for (int r = warp; r < 16 * NTW; r += nwarp) {
    const bool have = r < half_sine_rows(m);  // table rows beyond the half table: zeros
    for (int c = lane; c < 2 * kh; c += 32) {
      if (have) cp_async8(Bs + r * LDB + c, half + static_cast<i64>(r) * 2 * kh + c);
      else Bs[r * LDB + c] = 0.0;
    }
  }
  for (int i = tid; i < m; i += nth) cp_async8(Ss + i, sc + i);
  // padding rows of both A tiles, never overwritten (the table's padding columns are zero, but
  // 0 * garbage may be NaN)
  for (int buf = 0; buf < 2; ++buf) {
    double* As = Ab + buf * KA * LDA;
    for (int idx = tid; idx < (kh - P.ne) * TR; idx += nth) As[(P.ne + idx / TR) * LDA + idx % TR] = 0.0;
    for (int idx = tid; idx < (P.no4 - m / 2) * TR; idx += nth) As[(kh + m / 2 + idx / TR) * LDA + idx % TR] = 0.0;
  }
  int tile = blockIdx.x;
  if (tile < ntile) {
    const double* __restrict__ src = tile_src(tile);
    const unsigned ab_s = static_cast<unsigned>(__cvta_generic_to_shared(Ab));
    while (ik < m) issue_item(src, ab_s);
  }
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  const int r8 = lane >> 2, c4 = lane & 3, r0 = 16 * (warp >> 1), nb0 = (warp & 1) * NTW;
  for (int it = 0; tile < ntile; tile += gridDim.x, ++it) {
    // this tile's group was committed a round ago; the next tile's loads are issued between
    // the MMA steps below (one item per step) and committed after them
    const int buf = it & 1, next = tile + gridDim.x;
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    const double* __restrict__ nsrc = next < ntile ? tile_src(next) : nullptr;
    const unsigned an_s = static_cast<unsigned>(__cvta_generic_to_shared(Ab + (buf ^ 1) * KA * LDA));
    ik = warp;
    ic = 0;
    const double* As = Ab + buf * KA * LDA + r0 + r8;
    const double* Bw = Bs + (8 * nb0 + r8) * LDB + c4;
    double E[2][NTW][2], O[2][NTW][2];
#pragma unroll
    for (int a = 0; a < 2; ++a)
#pragma unroll
      for (int b = 0; b < NTW; ++b) E[a][b][0] = E[a][b][1] = O[a][b][0] = O[a][b][1] = 0.0;
#pragma unroll 2
    for (int ks = 0; ks < kh; ks += 4) {
      const double a0 = As[(ks + c4) * LDA], a1 = As[(ks + c4) * LDA + 8];
      if (nsrc && ik < m) issue_item(nsrc, an_s);
#pragma unroll
      for (int b = 0; b < NTW; ++b) {
        const double fb = Bw[8 * b * LDB + ks];
        dmma(E[0][b], a0, fb);
        dmma(E[1][b], a1, fb);
      }
    }
#pragma unroll 2
    for (int ks = 0; ks < P.no4; ks += 4) {
      const double a0 = As[(kh + ks + c4) * LDA], a1 = As[(kh + ks + c4) * LDA + 8];
      if (nsrc && ik < m) issue_item(nsrc, an_s);
#pragma unroll
      for (int b = 0; b < NTW; ++b) {
        const double fb = Bw[8 * b * LDB + kh + ks];
        dmma(O[0][b], a0, fb);
        dmma(O[1][b], a1, fb);
      }
    }
    if (nsrc)
      while (ik < m) issue_item(nsrc, an_s);
    asm volatile("cp.async.commit_group;\n" ::: "memory");
    // out(q) = sc_q (E + O), out(m-1-q) = sc_{m-1-q} (E - O) straight from the accumulators
    const int box = tile / P.tiles, t = tile - box * P.tiles;
    const int j0 = min(t * TR, m1 - TR);
    const int bx = box % P.nbox0, by = box / P.nbox0;
    const int qb = 8 * nb0 + 2 * c4;  // this thread's first output of n tile 0
    double* __restrict__ dst = e + bx * P.out_bs0 + by * P.out_bs1 + static_cast<i64>(j0 + r0 + r8) * P.out_stride;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      double* __restrict__ pq = dst + static_cast<i64>(8 * a) * P.out_stride + qb;
      double* __restrict__ pm = dst + static_cast<i64>(8 * a) * P.out_stride + (m - 1 - qb);
#pragma unroll
      for (int b = 0; b < NTW; ++b) {
        if (8 * (nb0 + b) + 7 < P.mh - 1) {  // warp-uniform: every output of the tile and its mirror exist
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            pq[8 * b + h] = Ss[qb + 8 * b + h] * (E[a][b][h] + O[a][b][h]);
            pm[-(8 * b + h)] = Ss[m - 1 - qb - 8 * b - h] * (E[a][b][h] - O[a][b][h]);
          }
        } else {
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int q = qb + 8 * b + h;
            if (q < P.mh) {
              pq[8 * b + h] = Ss[q] * (E[a][b][h] + O[a][b][h]);
              if (m - 1 - q != q) pm[-(8 * b + h)] = Ss[m - 1 - q] * (E[a][b][h] - O[a][b][h]);
            }
          }
        }
      }
    }
    __syncthreads();  // every warp is done with this A tile before the next round refills it
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
}

int strip_back_warps(int m1) {
  if (const char* ev = std::getenv("ASDSM_STRIP_BACK_NW")) return std::max(2, std::min(8, std::atoi(ev)));
  // rows per tile = 16 x warps: the fewest padded rows over 4..7 warps (ties to more warps)
  int best = 6;
  double waste = 1e30;
  for (int nw = 3; nw <= 7; ++nw) {
    const int tr = 16 * nw;
    if (m1 < tr) continue;
    const double w = static_cast<double>((m1 + tr - 1) / tr * tr) / m1;
    if (w <= waste) {
      waste = w;
      best = nw;
    }
  }
  return best;
}

size_t strip_back_smem(int m, int nw) {
  const int kh = half_sine_kh(m), no4 = ((m / 2) + 3) & ~3, ntw = (((m + 1) / 2 + 7) / 8 + 1) / 2;
  return sizeof(double) * (static_cast<size_t>(16 * ntw) * (2 * kh + 4) + ((m + 1) & ~1) +
                           2 * static_cast<size_t>(kh + no4) * (16 * nw + 4));
}
}  // namespace

void dmma_prepare() {  // (a 3-stage cp.async variant of the dense kernel measured slower on both
                       // m=102 and m=409 and was dropped)
  static bool done = false;
  if (done) return;
  done = true;
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(strip_back_kernel<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(strip_back_kernel<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
#define ASDSM_EO2_ATTR(B, C)                                                                                      \
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(dmma_eo2_kernel<B, C, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kEo2Smem))); \
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(dmma_eo2_kernel<B, C, 48>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(kEo2Smem)));
  ASDSM_EO2_ATTR(true, true)
  ASDSM_EO2_ATTR(true, false)
  ASDSM_EO2_ATTR(false, true)
  ASDSM_EO2_ATTR(false, false)
#undef ASDSM_EO2_ATTR
}

void launch_dmma_eo_transform(bool back, const double* in, double* out, const double* half, int m, i64 in_es,
                              i64 out_es, const GemmLines& L, cudaStream_t s) {
  const int kh = half_sine_kh(m), hr = half_sine_rows(m), mh = (m + 1) / 2;
  const double* sc = half + static_cast<i64>(hr) * 2 * kh;
  const i64 pb = (L.nlines + EP - 1) / EP;
  if (pb > 65535) throw AsdsmError(kUnsupported, "transform batch too large for the grid");
  const int nq = back ? mh : kh;
  // output tile width: 64, or 48 when that pads the nq outputs less (259-point slab axes: 130
  // outputs are 3 tiles either way, 144 against 192 columns of MMAs; ASDSM_EO2_Q=64 forces 64)
  const bool q48 = ((nq + 47) / 48) * 48 < ((nq + 63) / 64) * 64 && std::getenv("ASDSM_EO2_Q") == nullptr;
  const int eq = q48 ? 48 : 64;
  dim3 grid(static_cast<unsigned>((nq + eq - 1) / eq), static_cast<unsigned>(pb));
  const bool ci = in_es == 1;
#define ASDSM_EO2_LAUNCH(B, C)                                                                                   \
  do {                                                                                                           \
    if (q48) dmma_eo2_kernel<B, C, 48><<<grid, ENT2, kEo2Smem, s>>>(in, out, half, sc, m, kh, in_es, out_es, L);  \
    else dmma_eo2_kernel<B, C, 64><<<grid, ENT2, kEo2Smem, s>>>(in, out, half, sc, m, kh, in_es, out_es, L);      \
  } while (0)
  if (back) {
    if (ci) ASDSM_EO2_LAUNCH(true, true);
    else ASDSM_EO2_LAUNCH(true, false);
  } else {
    if (ci) ASDSM_EO2_LAUNCH(false, true);
    else ASDSM_EO2_LAUNCH(false, false);
  }
#undef ASDSM_EO2_LAUNCH
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

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

bool strip_back_supported(int m, int m1) {
  const int nt = ((m + 1) / 2 + 7) / 8;
  if (m < 56 || nt < 4 || nt > 6 || m1 < 64) return false;
  const int nw = strip_back_warps(m1);
  return m1 >= 16 * nw && strip_back_smem(m, nw) <= 220 * 1024;
}

void launch_strip_back(const double* modes, double* e, const double* half, int m, int m1, int nbox0, int nbox1,
                       i64 out_bs0, i64 out_bs1, i64 out_stride, cudaStream_t s) {
  const int nw = strip_back_warps(m1), tr = 16 * nw;
  StripBackArgs P{};
  P.m = m;
  P.m1 = m1;
  P.kh = half_sine_kh(m);
  P.mh = (m + 1) / 2;
  P.ne = (m + 1) / 2;
  P.no4 = ((m / 2) + 3) & ~3;
  P.tiles = (m1 + tr - 1) / tr;
  P.nbox0 = nbox0;
  P.nboxes = nbox0 * nbox1;
  P.out_bs0 = out_bs0;
  P.out_bs1 = out_bs1;
  P.out_stride = out_stride;
  const long long ntile = static_cast<long long>(nbox0) * nbox1 * P.tiles;
  if (ntile > 0x7fffffffLL) throw AsdsmError(kUnsupported, "strip back transform: too many tiles");
  // persistent: as many CTAs as are resident at once walk the tiles
  const size_t smem_q = strip_back_smem(m, nw);
  int per_sm = 1;
  if ((P.mh + 7) / 8 <= 4) ASDSM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, strip_back_kernel<2>, 64 * nw, smem_q));
  else ASDSM_CUDA_CHECK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, strip_back_kernel<3>, 64 * nw, smem_q));
  const long long grid = std::min<long long>(ntile, static_cast<long long>(kNumSms) * std::max(per_sm, 1));
  const size_t smem = strip_back_smem(m, nw);
  const int nt = (P.mh + 7) / 8;  // 4..6 (strip_back_supported): a warp pair covers 2 x 2 or 2 x 3 n tiles
  if (nt <= 4) strip_back_kernel<2><<<static_cast<unsigned>(grid), 64 * nw, smem, s>>>(modes, e, half, P);
  else strip_back_kernel<3><<<static_cast<unsigned>(grid), 64 * nw, smem, s>>>(modes, e, half, P);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
