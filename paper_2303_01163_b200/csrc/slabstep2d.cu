// One-launch 2D slab step (error mode, lines up to kPartMaxLine fine points).
//
// The reference solves the two anisotropic slab systems A_fc, A_cf with SparseLU
// (linsolve.cpp:58-66, solver.cpp:550-558), normalizes both solutions (solver.cpp:79-84),
// takes the cross values and clamped-spline corrections (solver.cpp:166-187, spline.cpp) and
// scatters the skeleton into the fine array.  Here a cluster of two CTAs does all of it in one
// launch, CTA a owning slab a (coarse along axis a):
//   P1  the residual on the slab's stations (compact copy kept by the residual passes), the
//       eigenvector blocks and the line-solve tables -> shared memory
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
#include "skel2d.cuh"

#include <cooperative_groups.h>

namespace asdsm_b200 {

namespace cg = cooperative_groups;

namespace {

constexpr int kStepThreads = 320;  // 10 warps: one mode line per warp for nc <= 10
constexpr int kStepWarps = kStepThreads / 32;
constexpr int kStepMaxNc = 24;
constexpr int kRecip = 5 * kStepMaxNc;  // per spline family: 1/hl, 1/hr, 1/dg (nc), 1/h, 1/(6h) (nc+1)

struct StepLayout {
  int NC, NF, PS;
  int st, md, wv, pt, cr1, cr2, nrm, ce1, ce2, stab, rcp, srhs, smm, sg1, sg2, red, total;
};

__host__ __device__ inline StepLayout step_layout(const MeshDev& m, int pstride) {
  StepLayout L{};
  L.NC = m.nc[0] > m.nc[1] ? m.nc[0] : m.nc[1];
  L.NF = m.nf[0] > m.nf[1] ? m.nf[0] : m.nf[1];
  L.PS = pstride;
  const int ncc = m.nc[0] * m.nc[1];
  int o = 0;
  auto take = [&](int n) {
    const int r = o;
    o += (n + 1) & ~1;  // keep 16-byte alignment of every region
    return r;
  };
  L.st = take(L.NC * L.NF);
  L.md = take(L.NC * L.NF);
  L.wv = take(2 * L.NC * L.NC);
  L.pt = take(L.NC * pstride);
  L.cr1 = take(ncc);
  L.cr2 = take(ncc);
  L.nrm = take(2);
  L.ce1 = take(ncc);
  L.ce2 = take(ncc);
  L.stab = take(2 * kSkelTabMax);
  L.rcp = take(2 * kRecip);
  L.srhs = take((m.nc[0] + m.nc[1]) * kStepMaxNc);
  L.smm = take((m.nc[0] + m.nc[1]) * (kStepMaxNc + 2));
  L.sg1 = take(m.nc[1] * 4 * (m.nc[0] + 1));
  L.sg2 = take(m.nc[0] * 4 * (m.nc[1] + 1));
  L.red = take(32);
  L.total = o;
  return L;
}

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

// C[nc][nf] = Amat[nc][nc] * B[nc][nf] (B, C in shared memory; MT = ceil(nc/8) row tiles,
// KS = ceil(nc/4) k steps of m8n8k4), warps over the 8-column tiles; returns the warp's sum of
// squares of C when kNorm.
template <int MT, int KS, bool kNorm>
__device__ __forceinline__ double small_gemm(const double* Amat, const double* B, double* C, int nc, int nf) {
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
  const int ntiles = (nf + 7) >> 3;
  for (int nt = warp; nt < ntiles; nt += kStepWarps) {
    const int n0 = nt * 8;
    double b[KS];
#pragma unroll
    for (int ks = 0; ks < KS; ++ks) {
      const int k = ks * 4 + c4;
      b[ks] = (k < nc && n0 + r8 < nf) ? B[k * nf + n0 + r8] : 0.0;
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
        if (row < nc && col < nf) {
          C[row * nf + col] = acc[mt][h];
          if (kNorm) ss += acc[mt][h] * acc[mt][h];
        }
      }
    }
  }
  return ss;
}

template <bool kNorm>
__device__ __forceinline__ double gemm_dispatch(const double* Amat, const double* B, double* C, int nc, int nf) {
  if (nc <= 4) return small_gemm<1, 1, kNorm>(Amat, B, C, nc, nf);
  if (nc <= 8) return small_gemm<1, 2, kNorm>(Amat, B, C, nc, nf);
  if (nc <= 12) return small_gemm<2, 3, kNorm>(Amat, B, C, nc, nf);
  if (nc <= 16) return small_gemm<2, 4, kNorm>(Amat, B, C, nc, nf);
  if (nc <= 20) return small_gemm<3, 5, kNorm>(Amat, B, C, nc, nf);
  return small_gemm<3, 6, kNorm>(Amat, B, C, nc, nf);
}

// One line of mode space (length n, in shared memory, in place) by one warp; T = this mode's
// SepSolver::part table (in shared memory).  Every lane runs exactly SEG steps: rows past its
// segment have pivot 0, so they stay 0 and decouple.
template <int SEG>
__device__ __forceinline__ void part_solve_line(double* line, const double* T, int n, int P, int last, double l,
                                                double r) {
  constexpr int M = SEG + 1;
  const int q = threadIdx.x & 31;
  const int R = P - 1;
  const bool full = q < P - 1;
  const int Li = full ? SEG : (q == P - 1 ? last : 0);
  const int base = q * M;
  double y[SEG];
#pragma unroll
  for (int t = 0; t < SEG; ++t) y[t] = t < Li ? line[base + t] : 0.0;
  const double fs = q < R ? line[base + M - 1] : 0.0;
  // pivots (shared, broadcast) are read straight into the chain: zero past the segment
  y[0] = y[0] * (Li > 0 ? T[0] : 0.0);
  double ylast = y[0];  // y of the segment's last row (static indices keep y in registers)
#pragma unroll
  for (int t = 1; t < SEG; ++t) {
    y[t] = (y[t] - l * y[t - 1]) * (t < Li ? T[t] : 0.0);
    if (t < Li) ylast = y[t];
  }
#pragma unroll
  for (int t = SEG - 2; t >= 0; --t) y[t] = y[t] - (r * (t < Li ? T[t] : 0.0)) * y[t + 1];
  const double ynext0 = __shfl_down_sync(0xffffffffu, y[0], 1);
  double rho = q < R ? fs - l * ylast - r * ynext0 : 0.0;
  double c1[5], c2[5];
#pragma unroll
  for (int lev = 0; lev < 5; ++lev) {
    c1[lev] = T[part_off_k1(SEG) + lev * 32 + q];
    c2[lev] = T[part_off_k2(SEG) + lev * 32 + q];
  }
#pragma unroll
  for (int lev = 0; lev < 5; ++lev) {
    const int s = 1 << lev;
    const double up = __shfl_up_sync(0xffffffffu, rho, s);
    const double dn = __shfl_down_sync(0xffffffffu, rho, s);
    if (q < R) {
      double v = rho;
      if (q - s >= 0) v = v - c1[lev] * up;
      if (q + s < R) v = v - c2[lev] * dn;
      rho = v;
    }
  }
  const double xs = q < R ? rho * T[part_off_ib(SEG) + q] : 0.0;

  double xl = __shfl_up_sync(0xffffffffu, xs, 1);
  if (q == 0) xl = 0.0;
  const double xr = full ? xs : 0.0;
  const double* g = T + (full ? part_off_g(SEG) : part_off_gl(SEG));
  const double* h = T + part_off_h(SEG);
#pragma unroll
  for (int t = 0; t < SEG; ++t) {  // all table reads before the first store (shared may alias)
    double v = y[t] - g[t] * xl;
    if (full) v = v - h[t] * xr;
    y[t] = v;
  }
#pragma unroll
  for (int t = 0; t < SEG; ++t)
    if (t < Li) line[base + t] = y[t];
  if (q < R) line[base + M - 1] = xs;
}

__device__ __forceinline__ void solve_dispatch(int seg, double* line, const double* T, int n, int P, int last, double l, double r) {
  switch (seg) {
#define ASDSM_SEG(S_) \
  case S_:            \
    part_solve_line<S_>(line, T, n, P, last, l, r); \
    break;
    ASDSM_SEG(2) ASDSM_SEG(4) ASDSM_SEG(8) ASDSM_SEG(12) ASDSM_SEG(16) ASDSM_SEG(20) ASDSM_SEG(24) ASDSM_SEG(28)
    ASDSM_SEG(32)
#undef ASDSM_SEG
    default:
      break;
  }
}

// segment index of fine index fi (1-based) on an axis with factor n: fi / n clamped to nc,
// without an integer division
__device__ __forceinline__ int seg_of(int fi, int n, float invn, int nc) {
  int c = __float2int_rd(__int2float_rn(fi) * invn);
  if ((c + 1) * n <= fi) ++c;
  else if (c * n > fi) --c;
  return c > nc ? nc : c;
}

__device__ __forceinline__ double seg_eval(const double* tab, const double* seg, int c, double x) {
  const double t = __dsub_rn(x, tab[c]);
  const double* s = seg + 4 * c;
  return __dadd_rn(s[0], __dmul_rn(t, __dadd_rn(s[1], __dmul_rn(t, __dadd_rn(s[2], __dmul_rn(t, s[3]))))));
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kStepThreads, 1)
    slabstep2d_kernel(SlabStep2DArgs A, DevState* S) {
  if (!S->active) return;  // same decision in both CTAs of the cluster
#ifdef ASDSM_STEP_TRACE
  long long T_[10] = {clock64(), 0, 0, 0, 0, 0, 0, 0, 0, 0};
#define STEP_STAMP(i) T_[i] = clock64()
#else
#define STEP_STAMP(i)
#endif
  cg::cluster_group cluster = cg::this_cluster();
  extern __shared__ __align__(16) double sm[];
  const MeshDev& m = A.m;
  const int PS = A.pstride[0] > A.pstride[1] ? A.pstride[0] : A.pstride[1];
  const StepLayout Lo = step_layout(m, PS);
  const int a = static_cast<int>(cluster.block_rank()), f = 1 - a;
  const int nc = m.nc[a], nf = m.nf[f];
  const int nc0 = m.nc[0], nc1 = m.nc[1], ncc = nc0 * nc1;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  double* st = sm + Lo.st;
  double* md = sm + Lo.md;
  double* sW = sm + Lo.wv;
  double* sV = sW + nc * nc;
  double* pt = sm + Lo.pt;
  double* stab = sm + Lo.stab;
  double* rcp = sm + Lo.rcp;
  // P1
  const double* rs = (S->cur ? A.sta1 : A.sta0) + (a == 0 ? 0 : static_cast<i64>(nc0) * m.nf[1]);
  // bulk loads: cp.async keeps every request in flight (a load -> shared store loop would
  // wait one L2 round trip per element)
  for (int i = tid; i < nc * nf; i += kStepThreads) cp_async8(st + i, rs + i);
  for (int i = tid; i < nc * nc; i += kStepThreads) {
    cp_async8(sW + i, A.W[a] + i);
    cp_async8(sV + i, A.V[a] + i);
  }
  for (int i = tid; i < nc * A.pstride[a]; i += kStepThreads) cp_async8(pt + i, A.part[a] + i);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  for (int fam = 0; fam < 2; ++fam) {  // spline tables and the reciprocals of their widths
    const int ncf = m.nc[fam], tl = (ncf + 2) + 5 * ncf;
    const double* src = A.sp_tab[fam];
    double* dt = stab + fam * kSkelTabMax;
    double* dr = rcp + fam * kRecip;
    for (int q = tid; q < tl; q += kStepThreads) cp_async8(dt + q, src + q);
    for (int q = tid; q < 5 * kStepMaxNc; q += kStepThreads) {
      const int kind = q / kStepMaxNc, i = q % kStepMaxNc;
      double v = 0.0;
      if (kind == 0 && i < ncf) v = 1.0 / __ldg(src + ncf + 2 + i);               // 1 / hl
      else if (kind == 1 && i < ncf) v = 1.0 / __ldg(src + 2 * ncf + 2 + i);      // 1 / hr
      else if (kind == 2 && i < ncf) v = 1.0 / __ldg(src + 4 * ncf + 2 + i);      // 1 / diag
      else if (kind >= 3 && i <= ncf) {
        const double h = __dsub_rn(__ldg(src + i + 1), __ldg(src + i));
        v = kind == 3 ? 1.0 / h : 1.0 / __dmul_rn(6.0, h);
      }
      dr[q] = v;
    }
  }
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  STEP_STAMP(1);
  // P2: md = W st
  gemm_dispatch<false>(sW, st, md, nc, nf);
  __syncthreads();
  STEP_STAMP(2);
  // P3
  for (int k = warp; k < nc; k += kStepWarps)
    solve_dispatch(A.pseg[a], md + k * nf, pt + k * A.pstride[a], nf, A.pP[a], A.plast[a], A.line_l[a], A.line_r[a]);
  __syncthreads();
  STEP_STAMP(3);
  // P4: sol = V md -> st, squared norm
  double ss = gemm_dispatch<true>(sV, md, st, nc, nf);
  double* red = sm + Lo.red;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_down_sync(0xffffffffu, ss, o);
  if (lane == 0) red[warp] = ss;
  __syncthreads();
  STEP_STAMP(4);
  // P5: exchange the norm and the cross values with the peer CTA
  double* nrm = sm + Lo.nrm;
  double* cr1 = sm + Lo.cr1;  // u_fc at the cross points (slab 1)
  double* cr2 = sm + Lo.cr2;  // u_cf at the cross points (slab 0)
  double* peer_nrm = cluster.map_shared_rank(nrm, 1 - a);
  double* peer_cr = cluster.map_shared_rank(a == 1 ? cr1 : cr2, 1 - a);
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < kStepWarps; ++w) t += red[w];
    nrm[a] = t;
    peer_nrm[a] = t;
  }
  for (int t = tid; t < ncc; t += kStepThreads) {
    const int I = t % nc0, J = t / nc0;
    double v;
    if (a == 1) v = st[J * nf + (I + 1) * m.n[0] - 1];  // u_fc(x = station I, J)
    else v = st[I * nf + (J + 1) * m.n[1] - 1];         // u_cf(I, y = station J)
    (a == 1 ? cr1 : cr2)[t] = v;
    peer_cr[t] = v;
  }
  cluster.sync();
  STEP_STAMP(5);
  const double ncf = sqrt(nrm[0]), nfc = sqrt(nrm[1]);
  if (a == 0 && tid == 0) {
    S->slab_norm[0] = ncf;
    S->slab_norm[1] = nfc;
    if (!(ncf > 0.0) || !(nfc > 0.0)) S->have_e = 0;
  }
  if (!(ncf > 0.0) || !(nfc > 0.0)) return;  // ZeroNormSolution: no correction this step
  const double ifc = 1.0 / nfc, icf = 1.0 / ncf;
  // P6: corrections at the cross points (error mode: the coin picks the slab), spline segments
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
  double* srhs = sm + Lo.srhs;  // [line][i], lines: nc1 along x then nc0 along y
  double* smm = sm + Lo.smm;    // [line][c]
  double* sg1 = sm + Lo.sg1;
  double* sg2 = sm + Lo.sg2;
  const int nlines = nc0 + nc1;
  auto yval = [&](int line, int c) -> double {
    if (line < nc1) return (c == 0 || c == nc0 + 1) ? 0.0 : ce1[(c - 1) + nc0 * line];
    const int I = line - nc1;
    return (c == 0 || c == nc1 + 1) ? 0.0 : ce2[I + nc0 * (c - 1)];
  };
  for (int t = tid; t < 2 * ncc; t += kStepThreads) {
    const int line = t < ncc ? t / nc0 : nc1 + (t - ncc) / nc1;
    const int i = t < ncc ? t % nc0 : (t - ncc) % nc1;
    const double* rr = rcp + (line < nc1 ? 0 : kRecip);
    srhs[line * kStepMaxNc + i] = __dsub_rn(__dmul_rn(__dsub_rn(yval(line, i + 2), yval(line, i + 1)), rr[kStepMaxNc + i]),
                                            __dmul_rn(__dsub_rn(yval(line, i + 1), yval(line, i)), rr[i]));
  }
  __syncthreads();
  for (int line = tid; line < nlines; line += kStepThreads) {
    const int ni = line < nc1 ? nc0 : nc1, n = ni + 2;
    const double* tab = stab + (line < nc1 ? 0 : kSkelTabMax);
    const double* rr = rcp + (line < nc1 ? 0 : kRecip);
    const double* w = tab + n + 2 * ni;
    const double* up = w + 2 * ni;
    double* rhs = srhs + line * kStepMaxNc;
    double* mm = smm + line * (kStepMaxNc + 2);
    for (int i = 1; i < ni; ++i) rhs[i] = __dsub_rn(rhs[i], __dmul_rn(w[i], rhs[i - 1]));
    mm[0] = 0.0;
    mm[n - 1] = 0.0;
    if (ni > 0) {
      mm[ni] = __dmul_rn(rhs[ni - 1], rr[2 * kStepMaxNc + ni - 1]);
      for (int i = ni - 1; i >= 1; --i)
        mm[i] = __dmul_rn(__dsub_rn(rhs[i - 1], __dmul_rn(up[i - 1], mm[i + 1])), rr[2 * kStepMaxNc + i - 1]);
    }
  }
  __syncthreads();
  for (int t = tid; t < nc1 * (nc0 + 1) + nc0 * (nc1 + 1); t += kStepThreads) {
    int line, c;
    if (t < nc1 * (nc0 + 1)) {
      line = t / (nc0 + 1);
      c = t % (nc0 + 1);
    } else {
      line = nc1 + (t - nc1 * (nc0 + 1)) / (nc1 + 1);
      c = (t - nc1 * (nc0 + 1)) % (nc1 + 1);
    }
    const double* x = stab + (line < nc1 ? 0 : kSkelTabMax);
    const double* rr = rcp + (line < nc1 ? 0 : kRecip);
    const double* mm = smm + line * (kStepMaxNc + 2);
    const double y0 = yval(line, c), y1 = yval(line, c + 1);
    const double h = __dsub_rn(x[c + 1], x[c]);
    double* seg = line < nc1 ? sg1 + line * 4 * (nc0 + 1) + 4 * c : sg2 + (line - nc1) * 4 * (nc1 + 1) + 4 * c;
    seg[0] = y0;
    seg[1] = __dsub_rn(__dmul_rn(__dsub_rn(y1, y0), rr[3 * kStepMaxNc + c]),
                       __dmul_rn(__dmul_rn(h, __dadd_rn(__dmul_rn(2.0, mm[c]), mm[c + 1])), 1.0 / 6.0));
    seg[2] = __dmul_rn(mm[c], 0.5);
    seg[3] = __dmul_rn(__dsub_rn(mm[c + 1], mm[c]), rr[4 * kStepMaxNc + c]);
  }
  __syncthreads();
  STEP_STAMP(6);
  // P7: skeleton write (skel2d_write_fast_kernel's arithmetic)
  const i64 Nx = m.nf[0];
  const double* tab0 = stab;
  const double* tab1 = stab + kSkelTabMax;
  const float invn0 = 1.0f / static_cast<float>(m.n[0]), invn1 = 1.0f / static_cast<float>(m.n[1]);
  if (a == 1) {  // lines along x at the y-stations: u_fc / nfc + spline, cross points (av + bv) - bv
    for (int J = 0; J < nc1; ++J) {
      const int j = (J + 1) * m.n[1] - 1;
      const int cj = seg_of(j + 1, m.n[1], invn1, nc1);
      const double xj = static_cast<double>(j + 1) * m.h[1];
      const double* s1 = sg1 + J * 4 * (nc0 + 1);
      const double* srow = st + J * nf;
      double* orow = A.out + Nx * j;
#pragma unroll 4
      for (int i = tid; i < m.nf[0]; i += kStepThreads) {
        const int fi = i + 1;
        const int c = seg_of(fi, m.n[0], invn0, nc0);
        const double ufc = srow[i] * ifc;
        const double av = __dadd_rn(ufc, seg_eval(tab0, s1, c, static_cast<double>(fi) * m.h[0]));
        double val = av;
        if (c * m.n[0] == fi && c >= 1) {  // an x-station: cross point
          const int I = c - 1;
          const double ucf = cr2[I + nc0 * J] * icf;
          const double bv = __dadd_rn(ucf, seg_eval(tab1, sg2 + I * 4 * (nc1 + 1), cj, xj));
          val = __dadd_rn(__dadd_rn(av, bv), -bv);
        }
        orow[i] = val;
      }
    }
  } else {  // lines along y at the x-stations (cross points are written by CTA 1)
    for (int I = 0; I < nc0; ++I) {
      const int i = (I + 1) * m.n[0] - 1;
      const double* s2 = sg2 + I * 4 * (nc1 + 1);
      const double* scol = st + I * nf;
#pragma unroll 4
      for (int j = tid; j < m.nf[1]; j += kStepThreads) {
        const int fj = j + 1;
        const int c = seg_of(fj, m.n[1], invn1, nc1);
        if (c * m.n[1] == fj && c >= 1 && c <= nc1) continue;  // a y-station: cross point
        const double ucf = scol[j] * icf;
        A.out[i + Nx * j] = __dadd_rn(ucf, seg_eval(tab1, s2, c, static_cast<double>(fj) * m.h[1]));
      }
    }
  }
#ifdef ASDSM_STEP_TRACE
  __syncthreads();
  STEP_STAMP(7);
  if (tid == 0)
    printf("STEPDBG cta %d load %lld tf %lld solve %lld back %lld xchg %lld ccspline %lld write %lld\n", a,
           T_[1] - T_[0], T_[2] - T_[1], T_[3] - T_[2], T_[4] - T_[3], T_[5] - T_[4], T_[6] - T_[5], T_[7] - T_[6]);
#endif
#undef STEP_STAMP
}

}  // namespace

bool slabstep2d_supported(const MeshDev& m, const SepSolver* slab) {
  if (m.dim != 2 || m.nc[0] > kStepMaxNc - 2 || m.nc[1] > kStepMaxNc - 2) return false;
  for (int a = 0; a < 2; ++a)
    if (slab[a].part == nullptr || slab[a].complex_modes) return false;
  const int ps = std::max(slab[0].part_stride, slab[1].part_stride);
  return sizeof(double) * static_cast<size_t>(step_layout(m, ps).total) <= 220 * 1024;
}

size_t slabstep2d_smem_bytes(const SlabStep2DArgs& A) {
  return sizeof(double) * static_cast<size_t>(step_layout(A.m, std::max(A.pstride[0], A.pstride[1])).total);
}

void slabstep2d_prepare() {
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(slabstep2d_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
}

void launch_slabstep2d(const SlabStep2DArgs& A, DevState* st, cudaStream_t s) {
  slabstep2d_kernel<<<2, kStepThreads, slabstep2d_smem_bytes(A), s>>>(A, st);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

}  // namespace asdsm_b200
