// 3D error-mode hole fill in ONE kernel per hole (fill_core, proj/src/solver.cpp:414-432, for the
// separable hole solver with diagonalized axes x, y and line axis t = axis 2).
//
// The hole rhs 0 - A_ff*skeleton lives on the hole's faces, so its forward transform is
// face-sparse (holes3d.cu explains the split into YA / XB / CH).  Per hole:
//   faces : ring values f from the skeleton, YA_f[t][l] = (Wy A_f(.,t))[l],
//           XB_f[t][k] = (Wx B_f(.,t))[k], CH_f = Wx C_f Wy^T     (pair sums, then DMMA dots)
//   lines : per mode pair (k,l) the Thomas solve along t of
//           fhat(t) = Wx[k][0] YA_0 + Wx[k][m-1] YA_1 + Wy[l][0] XB_0 + Wy[l][m-1] XB_1 (+ CH at t=0, m-1)
//   back  : per plane t, out = Vx X_t Vy^T as two DMMA GEMMs from shared memory.
// Every transform uses the even/odd split of the sine factor (plan.cpp half_sine_tables):
// V = D S, W = c S D^-1 and row m-1-i of S is (-1)^k times row i, so a back transform is
// E_i = sum_{k even} S[i][k] x_k, O_i = sum_{k odd} S[i][k] x_k over i < ceil(m/2) and
// out(i) = sc_i (E_i + O_i), out(m-1-i) = sc_{m-1-i} (E_i - O_i): half the MMAs of a dense V.
// The plane buffer keeps modes in even/odd order on both axes (row r(l), column c(k)):
//   step A (in place, a warp owns 8-row blocks): P[row][i] = sum_k X[row][k] Vx[i][k]
//   step B (per plane and j tile):               out[j][i] = sum_l Vy[j][l] P[l][i]  -> fine array
// Two schedules:
//   SYM    (central t stencil, whole hole in shared memory): forward sweep of every line, back
//          substitution in place (pivot tables streamed through a register pipeline), then the
//          back transform of every plane;
//   CAUSAL (backward time stencil: line_right == 0 -- the bidiagonal line has one pivot and no
//          back substitution): planes are produced in t order, TC planes at a time, the line
//          values ride in registers (thread (k, l0) owns the lines (k, l0 + G u)) -- any hole
//          depth; per chunk: dots -> line steps -> step A -> step B, the next chunk's pair sums
//          right behind step B (4 CTA barriers per chunk).
// Replaces the faces / Thomas / two transform-GEMM launches (a 1 GB mode buffer written and read
// twice at config 4) by one pass that writes every hole value once.
#include "holes3d.cuh"

#include <algorithm>
#include <cstdlib>
#include <vector>

namespace asdsm_b200 {

namespace {

constexpr int kH3Threads = 512;
constexpr int kH3Warps = kH3Threads / 32;
constexpr int kCausalLines = 8;  // CAUSAL: (k,l) lines per thread (mx*my <= 4096)
constexpr int kSymLines = 2;     // SYM: lines per thread (mx*my <= 1024)
#ifndef ASDSM_H3_PIPE
#define ASDSM_H3_PIPE 8
#endif
constexpr int kPipe = ASDSM_H3_PIPE;  // SYM: t steps per pivot-table load batch

__device__ __forceinline__ void dmma884(double (&d)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d[0]), "+d"(d[1])
               : "d"(a), "d"(b));
}

struct Geo {
  int ox, oy, oz;
};

// 0 - row_dot(p, skeleton) at hole point (i,j,t): CSR column order (fdm.cpp:110-117), as ring3
// in holes3d.cu
__device__ __forceinline__ double ring_val(const double* __restrict__ e, const Hole3DFusedArgs& A, const Geo& h, int i,
                                           int j, int t) {
  const Stencil& st = A.st;
  const i64 sy = A.nf[0], sz = static_cast<i64>(A.nf[0]) * A.nf[1];
  const i64 p = (h.ox + i) + (h.oy + j) * sy + (h.oz + t) * sz;
  double acc = 0.0;
  if (t == 0 && h.oz > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[2], __ldg(e + p - sz)));
  if (j == 0 && h.oy > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[1], __ldg(e + p - sy)));
  if (i == 0 && h.ox > 0) acc = __dadd_rn(acc, __dmul_rn(st.left[0], __ldg(e + p - 1)));
  if (i == A.m[0] - 1 && h.ox + A.m[0] < A.nf[0] && st.has_right[0]) acc = __dadd_rn(acc, __dmul_rn(st.right[0], __ldg(e + p + 1)));
  if (j == A.m[1] - 1 && h.oy + A.m[1] < A.nf[1] && st.has_right[1]) acc = __dadd_rn(acc, __dmul_rn(st.right[1], __ldg(e + p + sy)));
  if (t == A.m[2] - 1 && h.oz + A.m[2] < A.nf[2] && st.has_right[2]) acc = __dadd_rn(acc, __dmul_rn(st.right[2], __ldg(e + p + sz)));
  return __dsub_rn(0.0, acc);
}

// Half-table view of one diagonalized axis in shared memory: S rows i < he (stride sh, column
// c(k) = k/2 for even k, khe + k/2 for odd k), then sc[m] and ci[m] = (2/(m+1))/sc.
struct HalfTab {
  const double* S;
  const double* sc;
  const double* ci;
  int m, he, ho, khe, sh;
  __device__ __forceinline__ int col(int k) const { return (k & 1) ? khe + (k >> 1) : (k >> 1); }
  __device__ __forceinline__ double s0(int k) const { return S[col(k)]; }  // S[0][k]
};

__device__ __forceinline__ HalfTab half_tab(const double* base, const H3Axis& a) {
  HalfTab t;
  t.S = base;
  t.sc = base + a.hrow * a.sh;
  t.ci = t.sc + a.m;
  t.m = a.m;
  t.he = a.he;
  t.ho = a.ho;
  t.khe = a.khe;
  t.sh = a.sh;
  return t;
}

// Forward transforms of a batch of nv vectors (length T.m; value i of vector v = in(v, i)) on
// one axis: out(v, k) = sum_i W[k][i] v_i = sum_{i < he} S[i][k] h_{k&1}(i) with the pair sums
// h+/-(i) = ci_i v_i +/- ci_{m-1-i} v_{m-1-i} (i < ho; the middle point alone), built in Hb
// ([nv][2][he]) first (fwd_pairs), then the dots (fwd_dots_mma).  The two phases are separated
// by a barrier; the caller syncs after.
template <typename In>
__device__ __forceinline__ void fwd_pairs(const HalfTab& T, int nv, In in, double* Hb) {
  const int he = T.he, m = T.m;
  for (int q = threadIdx.x; q < nv * he; q += kH3Threads) {
    const int v = q / he, i = q - v * he;
    const double a = T.ci[i] * in(v, i);
    double hp = a, hm = a;
    if (i < T.ho) {
      const double b = T.ci[m - 1 - i] * in(v, m - 1 - i);
      hp = a + b;
      hm = a - b;
    }
    Hb[v * 2 * he + i] = hp;
    Hb[v * 2 * he + he + i] = hm;
  }
}
// The dots of the forward transforms on the DMMA pipe: per parity class the [modes x he] x [he x nv] product
// out(v, k) = sum_i S[i][c(k)] h_{k&1}(v, i), one (parity, 8 modes, 8 vectors) tile per task
// (tasks are dealt to warps by the caller: fwd_mma_tasks of them).  Rows i >= he of S are zero
// in the table and the h operand is masked there, so the padded K steps add exact zeros.
__device__ __forceinline__ int fwd_mma_tasks(const HalfTab& T, int nv) { return 2 * ((T.he + 7) >> 3) * ((nv + 7) >> 3); }
template <typename Out>
__device__ __forceinline__ void fwd_dots_mma(const HalfTab& T, int nv, const double* Hb, int task, Out out) {
  const int lane = threadIdx.x & 31, ar = lane >> 2, ak = lane & 3;
  const int he = T.he;
  const int nmt = (he + 7) >> 3, nnt = (nv + 7) >> 3;
  const int par = task / (nmt * nnt), rem = task - par * nmt * nnt, mt = rem / nnt, nt = rem - mt * nnt;
  const int v = 8 * nt + ar;  // this lane's B column (vector)
  const bool vok = v < nv;
  const double* hv = Hb + (vok ? (v * 2 + par) * he : 0);
  const double* sa = T.S + (par ? T.khe : 0) + 8 * mt + ar;
  double acc[2] = {0.0, 0.0};
  const int ksteps = (he + 3) >> 2;
  for (int kk = 0; kk < ksteps; ++kk) {
    const int i = 4 * kk + ak;
    const double a = sa[i * T.sh];
    const double b = (vok && i < he) ? hv[i] : 0.0;
    dmma884(acc, a, b);
  }
  const int k = 2 * (8 * mt + ar) + par;  // mode of this lane's accumulator row
  if (k < T.m) {
#pragma unroll
    for (int hh = 0; hh < 2; ++hh) {
      const int v2 = 8 * nt + 2 * ak + hh;
      if (v2 < nv) out(v2, k, acc[hh]);
    }
  }
}
template <typename Out>
__device__ __forceinline__ void fwd_dots_all(const HalfTab& T, int nv, const double* Hb, Out out) {
  const int nt = fwd_mma_tasks(T, nv);
  for (int task = threadIdx.x >> 5; task < nt; task += kH3Warps) fwd_dots_mma(T, nv, Hb, task, out);
}

// The MMA loops of the back transform with the tile count as a compile-time constant: a runtime
// `if (j < n)` around each mma.sync costs a predicate, its own address arithmetic and a
// WARPSYNC per MMA (8 instructions per DMMA in the profile); these are one LDS per operand.
// step A: a = this lane's row of X (even then odd mode columns), b = rows of the half table
template <int NT>
__device__ __forceinline__ void step_a_mma(const double* Ar, const double* Sb, int sh, int khe, int kev, int kod,
                                           double (&ae)[4][2], double (&ao)[4][2]) {
  for (int kk = 0; kk < kev; ++kk) {
    const double a = Ar[4 * kk];
    const double* b = Sb + 4 * kk;
#pragma unroll
    for (int j = 0; j < NT; ++j) dmma884(ae[j], a, b[8 * j * sh]);
  }
  for (int kk = 0; kk < kod; ++kk) {
    const double a = Ar[khe + 4 * kk];
    const double* b = Sb + khe + 4 * kk;
#pragma unroll
    for (int j = 0; j < NT; ++j) dmma884(ao[j], a, b[8 * j * sh]);
  }
}
// step B: a = rows of the y half table, b = rows of the plane (8-column tiles)
template <int NT>
__device__ __forceinline__ void step_b_mma(const double* Ay, const double* Pk0, int skx, int khe, int kev, int kod,
                                           double (&ae)[4][2], double (&ao)[4][2]) {
  for (int kk = 0; kk < kev; ++kk) {
    const double a = Ay[4 * kk];
    const double* Pk = Pk0 + 4 * kk * skx;
#pragma unroll
    for (int j = 0; j < NT; ++j) dmma884(ae[j], a, Pk[8 * j]);
  }
  for (int kk = 0; kk < kod; ++kk) {
    const double a = Ay[khe + 4 * kk];
    const double* Pk = Pk0 + (khe + 4 * kk) * skx;
#pragma unroll
    for (int j = 0; j < NT; ++j) dmma884(ao[j], a, Pk[8 * j]);
  }
}

// Back transform of `np` consecutive planes held in X (plane stride rp*skx; row r(l), column
// c(k); finite everywhere, zero where no mode lives), planes t0.. of the hole.
__device__ void back_planes(double* X, int np, int t0, const HalfTab& Tx, const HalfTab& Ty, const Hole3DFusedArgs& A,
                            const Geo& h, double* __restrict__ e, long long* tr = nullptr) {
  const int mx = A.m[0], my = A.m[1];
  const int skx = A.lay.skx, rp = A.lay.rp;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ar = lane >> 2, ak = lane & 3;
  // ---- step A: every row of the chunk, even/odd modes k -> points i (natural order), in place
  {
    const int ntx = (Tx.he + 7) >> 3;  // <= 4
    const int kev = Tx.khe >> 2, kod = (A.lay.kxo) >> 2;
    const int rows = np * rp;
    const int nrb = (rows + 7) >> 3;
    for (int rb = warp; rb < nrb; rb += kH3Warps) {
      double* Ar = X + static_cast<i64>(rb) * 8 * skx + ar * skx;
      double ae[4][2], ao[4][2];
#pragma unroll
      for (int j = 0; j < 4; ++j) ae[j][0] = ae[j][1] = ao[j][0] = ao[j][1] = 0.0;
      {
        const double* Sb = Tx.S + ar * Tx.sh + ak;
        switch (ntx) {
          case 4: step_a_mma<4>(Ar + ak, Sb, Tx.sh, Tx.khe, kev, kod, ae, ao); break;
          case 3: step_a_mma<3>(Ar + ak, Sb, Tx.sh, Tx.khe, kev, kod, ae, ao); break;
          case 2: step_a_mma<2>(Ar + ak, Sb, Tx.sh, Tx.khe, kev, kod, ae, ao); break;
          default: step_a_mma<1>(Ar + ak, Sb, Tx.sh, Tx.khe, kev, kod, ae, ao); break;
        }
      }
      __syncwarp();
      if (rb * 8 + ar < rows) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          if (j >= ntx) break;
          const int i0 = 8 * j + 2 * ak;
          if (i0 + 1 < Tx.he && !(mx & 1)) {  // both points and both mirrors: two 16-byte stores
            const int im1 = mx - 2 - i0;
            *reinterpret_cast<double2*>(Ar + i0) =
                make_double2(Tx.sc[i0] * (ae[j][0] + ao[j][0]), Tx.sc[i0 + 1] * (ae[j][1] + ao[j][1]));
            *reinterpret_cast<double2*>(Ar + im1) =
                make_double2(Tx.sc[im1] * (ae[j][1] - ao[j][1]), Tx.sc[im1 + 1] * (ae[j][0] - ao[j][0]));
            continue;
          }
#pragma unroll
          for (int hh = 0; hh < 2; ++hh) {
            const int i = i0 + hh;
            if (i < Tx.he) {
              const int im = mx - 1 - i;
              Ar[i] = Tx.sc[i] * (ae[j][hh] + ao[j][hh]);
              if (im != i) Ar[im] = Tx.sc[im] * (ae[j][hh] - ao[j][hh]);
            }
          }
        }
      }
    }
  }
  __syncthreads();
  if (tr) *tr = clock64();
  // ---- step B: out[t][j][i] = sum_l Vy[j][l] P[t][l][i] (rows of P in even/odd order)
  const i64 sy = A.nf[0], sz = static_cast<i64>(A.nf[0]) * A.nf[1];
  const int nty = (Ty.he + 7) >> 3;
  const int ntf = (mx + 7) >> 3;  // <= 8
  const int kev = Ty.khe >> 2, kod = A.lay.kyo >> 2;
  const int ntask = np * nty * ((ntf + 3) >> 2);
  for (int task = warp; task < ntask; task += kH3Warps) {
    const int nq = (ntf + 3) >> 2;
    const int pl = task / (nty * nq), rem = task - pl * nty * nq, jt = rem / nq, n0 = 4 * (rem - jt * nq);
    const double* P = X + static_cast<i64>(pl) * rp * skx + ar + 8 * n0;
    const double* Ay = Ty.S + (8 * jt + ar) * Ty.sh + ak;
    const int nn = min(4, ntf - n0);
    double ae[4][2], ao[4][2];
#pragma unroll
    for (int j = 0; j < 4; ++j) ae[j][0] = ae[j][1] = ao[j][0] = ao[j][1] = 0.0;
    switch (nn) {
      case 4: step_b_mma<4>(Ay, P + ak * skx, skx, Ty.khe, kev, kod, ae, ao); break;
      case 3: step_b_mma<3>(Ay, P + ak * skx, skx, Ty.khe, kev, kod, ae, ao); break;
      case 2: step_b_mma<2>(Ay, P + ak * skx, skx, Ty.khe, kev, kod, ae, ao); break;
      default: step_b_mma<1>(Ay, P + ak * skx, skx, Ty.khe, kev, kod, ae, ao); break;
    }
    const int jr = 8 * jt + ar;
    if (jr < Ty.he) {
      const int jm = my - 1 - jr;
      const double s0 = Ty.sc[jr], s1 = Ty.sc[jm];
      double* d0 = e + h.ox + (h.oy + jr) * sy + (h.oz + t0 + pl) * sz;
      double* d1 = e + h.ox + (h.oy + jm) * sy + (h.oz + t0 + pl) * sz;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (j >= nn) break;
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int i = 8 * (n0 + j) + 2 * ak + hh;
          if (i < mx) {
            d0[i] = s0 * (ae[j][hh] + ao[j][hh]);
            if (jm != jr) d1[i] = s1 * (ae[j][hh] - ao[j][hh]);
          }
        }
      }
    }
  }
}

// z face t_face (x/y-face points excluded) -> CH[l][k] = (Wx C Wy^T)(k, l); F ([j][i]), G ([j][k])
// and Hb are scratch.
__device__ void zface_transform(const double* __restrict__ e, const Hole3DFusedArgs& A, const Geo& h, int tface,
                                double* F, double* G, double* Hb, double* CH, const HalfTab& Tx, const HalfTab& Ty) {
  const int mx = A.m[0], my = A.m[1];
  for (int q = threadIdx.x; q < mx * my; q += kH3Threads) {
    const int i = q % mx, j = q / mx;
    F[q] = (i > 0 && i < mx - 1 && j > 0 && j < my - 1) ? ring_val(e, A, h, i, j, tface) : 0.0;
  }
  __syncthreads();
  fwd_pairs(Tx, my, [&](int v, int i) { return F[v * mx + i]; }, Hb);  // rows C(., j)
  __syncthreads();
  fwd_dots_all(Tx, my, Hb, [&](int v, int k, double x) { G[v * mx + k] = x; });
  __syncthreads();
  fwd_pairs(Ty, mx, [&](int v, int j) { return G[j * mx + v]; }, Hb);  // columns G(., k)
  __syncthreads();
  fwd_dots_all(Ty, mx, Hb, [&](int v, int l, double x) { CH[l * mx + v] = x; });
  __syncthreads();
}

// NL: CAUSAL line slots per thread (5 covers config 4's 50 x 50 modes on 500 threads; the line
// values live in registers across the GEMM phases, so unused slots cost spills)
template <bool CAUSAL, int NL = kCausalLines>
__global__ void __launch_bounds__(kH3Threads, 1)
    hole3d_fused_kernel(double* __restrict__ e, Hole3DFusedArgs A, const DevState* S) {
  if (!S->active || !S->have_e) return;
  extern __shared__ __align__(16) double sm[];
  const int mx = A.m[0], my = A.m[1], mt = A.m[2];
  const H3Layout& L = A.lay;
  const int skx = L.skx, rp = L.rp;
  const int tid = threadIdx.x;
  // tables (zero padded on the host) -> shared
  for (int q = tid; q < L.ntx; q += kH3Threads) cp_async8(sm + L.tx + q, A.Hx + q);
  for (int q = tid; q < L.nty; q += kH3Threads) cp_async8(sm + L.ty + q, A.Hy + q);
  asm volatile("cp.async.commit_group;\n" ::: "memory");
  const HalfTab Tx = half_tab(sm + L.tx, A.ax), Ty = half_tab(sm + L.ty, A.ay);
  double* X = sm + L.x;
  int b = blockIdx.x;
  Geo h;
  {
    const int hx = b % A.nbox[0];
    b /= A.nbox[0];
    const int hy = b % A.nbox[1];
    const int hz = b / A.nbox[1];
    h.ox = hx * A.n[0];
    h.oy = hy * A.n[1];
    h.oz = hz * A.n[2];
  }
  const int ncombo = mx * my;
  const i64 ps = static_cast<i64>(rp) * skx;  // plane stride
  const double lft = A.line_left;
  auto rowof = [&](int l) { return (l & 1) ? Ty.khe + (l >> 1) : (l >> 1); };
  // The x-face terms enter every line as Wx[k][0] YA_0 + Wx[k][m-1] YA_1 = S0x[k] YApm[k&1] with
  // YApm = Wy (ci_0 A_0 +/- ci_{mx-1} A_1) -- the two faces are combined before the transform
  // (and likewise the y faces: S0y[l] XBpm[l&1]).
  // (read after the table copies land)
  auto face_weights = [&](double& cx0, double& cx1, double& cy0, double& cy1) {
    cx0 = Tx.ci[0];
    cx1 = mx > 1 ? Tx.ci[mx - 1] : 0.0;
    cy0 = Ty.ci[0];
    cy1 = my > 1 ? Ty.ci[my - 1] : 0.0;
  };
  if (!CAUSAL) {
#ifdef ASDSM_H3_TRACE
    long long q0 = clock64(), q1 = 0, q2 = 0, q3 = 0;
#define H3S(v) v = clock64()
#else
#define H3S(v)
#endif
    double* YA = sm + L.faces;      // [2 (+/-)][mt][my]
    double* XB = YA + 2 * mt * my;  // [2][mt][mx]
    double* CH = XB + 2 * mt * mx;  // [2][my][mx]
    double* FA = X;                 // [2][mt][my]  x faces (all j, t), scratch in the plane region
    double* FB = FA + 2 * mt * my;  // [2][mt][mx]  y faces (x-face points excluded)
    double* H1 = FB + 2 * mt * mx;  // pair sums of the YA batch
    double* H2 = H1 + 2 * mt * 2 * Ty.he;
    for (int q = tid; q < 2 * mt * my; q += kH3Threads) {
      const int f = q / (mt * my), r = q - f * mt * my, t = r / my, j = r - t * my;
      FA[q] = (f == 0 || mx > 1) ? ring_val(e, A, h, f == 0 ? 0 : mx - 1, j, t) : 0.0;
    }
    for (int q = tid; q < 2 * mt * mx; q += kH3Threads) {
      const int f = q / (mt * mx), r = q - f * mt * mx, t = r / mx, i = r - t * mx;
      FB[q] = ((f == 0 || my > 1) && i > 0 && i < mx - 1) ? ring_val(e, A, h, i, f == 0 ? 0 : my - 1, t) : 0.0;
    }
    asm volatile("cp.async.wait_group 0;\n" ::: "memory");
    __syncthreads();
    double cx0, cx1, cy0, cy1;
    face_weights(cx0, cx1, cy0, cy1);
    // vector v = sign * mt + t
    fwd_pairs(Ty, 2 * mt, [&](int v, int j) {
      const int sg = v >= mt, t = v - sg * mt;
      const double a0 = cx0 * FA[t * my + j], a1 = cx1 * FA[mt * my + t * my + j];
      return sg ? a0 - a1 : a0 + a1;
    }, H1);
    fwd_pairs(Tx, 2 * mt, [&](int v, int i) {
      const int sg = v >= mt, t = v - sg * mt;
      const double b0 = cy0 * FB[t * mx + i], b1 = cy1 * FB[mt * mx + t * mx + i];
      return sg ? b0 - b1 : b0 + b1;
    }, H2);
    __syncthreads();
    fwd_dots_all(Ty, 2 * mt, H1, [&](int v, int l, double x) { YA[v * my + l] = x; });
    fwd_dots_all(Tx, 2 * mt, H2, [&](int v, int k, double x) { XB[v * mx + k] = x; });
    __syncthreads();
    double* G = X + mx * my;
    double* HZ = G + mx * my;
    H3S(q1);
    zface_transform(e, A, h, 0, X, G, HZ, CH, Tx, Ty);
    if (mt > 1) zface_transform(e, A, h, mt - 1, X, G, HZ, CH + my * mx, Tx, Ty);
    else
      for (int q = tid; q < mx * my; q += kH3Threads) CH[my * mx + q] = 0.0;
    for (int q = tid; q < L.xsize; q += kH3Threads) X[q] = 0.0;
    __syncthreads();
#ifdef ASDSM_H3_TRACE
    const long long q1b = clock64();
#endif
    // line solves: lines c = tid + u * threads; pivot tables streamed kPipe steps ahead
    int kq[kSymLines], lq[kSymLines];
    bool ok[kSymLines];
    double* xp[kSymLines];
    const double* pv[kSymLines];
    double y[kSymLines], sx[kSymLines], sy[kSymLines];
#pragma unroll
    for (int u = 0; u < kSymLines; ++u) {
      const int c = tid + u * kH3Threads;
      ok[u] = c < ncombo;
      const int cc = ok[u] ? c : 0;
      kq[u] = cc % mx;
      lq[u] = cc / mx;
      xp[u] = X + rowof(lq[u]) * skx + Tx.col(kq[u]);
      pv[u] = A.ipiv + cc;
      sx[u] = Tx.s0(kq[u]);
      sy[u] = Ty.s0(lq[u]);
      y[u] = 0.0;
    }
    double cur[kSymLines][kPipe], nxt[kSymLines][kPipe];
#pragma unroll
    for (int u = 0; u < kSymLines; ++u)
#pragma unroll
      for (int q = 0; q < kPipe; ++q) cur[u][q] = (ok[u] && q < mt) ? __ldg(pv[u] + static_cast<i64>(q) * ncombo) : 0.0;
    for (int t0 = 0; t0 < mt; t0 += kPipe) {
#pragma unroll
      for (int u = 0; u < kSymLines; ++u)
#pragma unroll
        for (int q = 0; q < kPipe; ++q)
          nxt[u][q] = (ok[u] && t0 + kPipe + q < mt) ? __ldg(pv[u] + static_cast<i64>(t0 + kPipe + q) * ncombo) : 0.0;
#pragma unroll
      for (int q = 0; q < kPipe; ++q) {
        const int t = t0 + q;
        if (t < mt) {
#pragma unroll
          for (int u = 0; u < kSymLines; ++u) {
            if (!ok[u]) continue;
            const int k = kq[u], l = lq[u];
            double f = sx[u] * YA[((k & 1) * mt + t) * my + l];
            f = fma(sy[u], XB[((l & 1) * mt + t) * mx + k], f);
            if (t == 0) f += CH[l * mx + k];
            if (t == mt - 1 && mt > 1) f += CH[my * mx + l * mx + k];
            y[u] = (t == 0) ? f * cur[u][q] : (f - lft * y[u]) * cur[u][q];
            xp[u][t * ps] = y[u];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kSymLines; ++u)
#pragma unroll
        for (int q = 0; q < kPipe; ++q) cur[u][q] = nxt[u][q];
    }
    // back substitution x_t = y_t - cp_t x_{t+1}, t = mt-2 .. 0, in batches of kPipe
#pragma unroll
    for (int u = 0; u < kSymLines; ++u) pv[u] = A.cp + (ok[u] ? tid + u * kH3Threads : 0);
    const int nb = (mt - 1 + kPipe - 1) / kPipe;
#pragma unroll
    for (int u = 0; u < kSymLines; ++u)
#pragma unroll
      for (int q = 0; q < kPipe; ++q)
        cur[u][q] = (ok[u] && mt - 2 - q >= 0) ? __ldg(pv[u] + static_cast<i64>(mt - 2 - q) * ncombo) : 0.0;
    for (int bi = 0; bi < nb; ++bi) {
      const int top = mt - 2 - bi * kPipe;
#pragma unroll
      for (int u = 0; u < kSymLines; ++u)
#pragma unroll
        for (int q = 0; q < kPipe; ++q)
          nxt[u][q] = (ok[u] && top - kPipe - q >= 0) ? __ldg(pv[u] + static_cast<i64>(top - kPipe - q) * ncombo) : 0.0;
#pragma unroll
      for (int q = 0; q < kPipe; ++q) {
        const int t = top - q;
        if (t >= 0) {
#pragma unroll
          for (int u = 0; u < kSymLines; ++u) {
            if (!ok[u]) continue;
            y[u] = xp[u][t * ps] - cur[u][q] * y[u];
            xp[u][t * ps] = y[u];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < kSymLines; ++u)
#pragma unroll
        for (int q = 0; q < kPipe; ++q) cur[u][q] = nxt[u][q];
    }
    __syncthreads();
    H3S(q2);
    back_planes(X, mt, 0, Tx, Ty, A, h, e);
#ifdef ASDSM_H3_TRACE
    __syncthreads();
    q3 = clock64();
    if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == 500))
      printf("H3SYM blk %d faces %lld zfaces %lld sweeps %lld back %lld\n", blockIdx.x, q1 - q0, q1b - q1, q2 - q1b,
             q3 - q2);
#endif
#undef H3S
    return;
  }
  // ---------------- CAUSAL: planes in t order, TC at a time
  const int TC = L.tc;
  const int nring = 2 * my + 2 * mx;   // per plane: A0[my] A1[my] B0[mx] B1[mx]
  double* CH0 = sm + L.faces;          // [my][mx]
  double* V = CH0 + my * mx;           // [TC][nring] YA+ YA- XB+ XB- of the chunk
  double* HB = V + TC * nring;         // pair sums: [TC][2][2 he_y] then [TC][2][2 he_x]
  double* HBx = HB + TC * 4 * Ty.he;
  asm volatile("cp.async.wait_group 0;\n" ::: "memory");
  __syncthreads();
  double cx0, cx1, cy0, cy1;
  face_weights(cx0, cx1, cy0, cy1);
  zface_transform(e, A, h, 0, X, X + mx * my, X + 2 * mx * my, CH0, Tx, Ty);
  for (int q = tid; q < L.xsize; q += kH3Threads) X[q] = 0.0;
  // line state: thread (k, l0) = (tid % mx, tid / mx) owns the lines (k, l0 + G u), u < U, G even:
  // its lines share k, the l parity, the x-face term's address and sit G/2 plane rows apart, so a
  // line step is two loads, three flops and a store at constant offsets
  const int LG = L.lg;
  const int tk = tid % mx, tl0 = tid / mx;
  int nlines = 0;
  if (tl0 < LG && tl0 < my) nlines = min(L.lu, (my - tl0 + LG - 1) / LG);
  double yv[NL];
#pragma unroll
  for (int u = 0; u < NL; ++u) yv[u] = 0.0;
  // Ring values from raw skeleton values staged through shared memory one chunk ahead
  // (cp.async: no registers wait on the loads).  Per plane: XL[j] = e(ox-1, oy+j), XR[j] =
  // e(ox+mx, oy+j), YL[i] = e(ox+i, oy-1), YR[i] = e(ox+i, oy+my); plane 0 also needs the
  // values below the hole at the face points (RZ, same layout as the ring vectors).  Same
  // terms and order as ring_val, so the values are bitwise the same.
  double* RAW = HBx + TC * 4 * Tx.he;  // [2][TC][nring]
  double* RZ = RAW + 2 * TC * nring;   // [nring]
  const Stencil& stn = A.st;
  const i64 esy = A.nf[0], esz = static_cast<i64>(A.nf[0]) * A.nf[1];
  const bool hxl = h.ox > 0, hxr = h.ox + mx < A.nf[0] && stn.has_right[0];
  const bool hyl = h.oy > 0, hyr = h.oy + my < A.nf[1] && stn.has_right[1];
  // thread r < nring owns ring position r of every plane: its source offset within a plane and
  // whether the neighbour exists are fixed for the kernel, a chunk is TC copies a plane apart
  i64 rsrc = 0;
  bool rok = false;
  if (tid < nring) {
    if (tid < 2 * my) {
      const int f = tid / my, j = tid - f * my;
      rok = f == 0 ? hxl : hxr;
      rsrc = (f == 0 ? h.ox - 1 : h.ox + mx) + (h.oy + j) * esy;
    } else {
      const int r2 = tid - 2 * my, f = r2 / mx, i = r2 - f * mx;
      rok = f == 0 ? hyl : hyr;
      rsrc = (h.ox + i) + (f == 0 ? h.oy - 1 : h.oy + my) * esy;
    }
    rsrc += h.oz * esz;
  }
  auto stage_raw = [&](int c) {
    const int t0c = c * TC;
    if (t0c < mt && tid < nring) {
      double* dst = RAW + (c & 1) * TC * nring + tid;
      const int npc = min(TC, mt - t0c);
      const double* src = e + rsrc + t0c * esz;
      for (int tt = 0; tt < npc; ++tt) {
        if (rok) cp_async8(dst + tt * nring, src + tt * esz);
        else dst[tt * nring] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\n" ::: "memory");
  };
  auto ring_raw = [&](const double* rp, double ez, int i, int j, bool t0) -> double {
    double acc = 0.0;
    if (t0 && h.oz > 0) acc = __dadd_rn(acc, __dmul_rn(stn.left[2], ez));
    if (j == 0 && hyl) acc = __dadd_rn(acc, __dmul_rn(stn.left[1], rp[2 * my + i]));
    if (i == 0 && hxl) acc = __dadd_rn(acc, __dmul_rn(stn.left[0], rp[j]));
    if (i == mx - 1 && hxr) acc = __dadd_rn(acc, __dmul_rn(stn.right[0], rp[my + j]));
    if (j == my - 1 && hyr) acc = __dadd_rn(acc, __dmul_rn(stn.right[1], rp[2 * my + mx + i]));
    return __dsub_rn(0.0, acc);
  };
  // values below the hole at the face points of plane 0 (x faces all j, y faces all i)
  if (h.oz > 0)
    for (int r = tid; r < nring; r += kH3Threads) {
      int i, j;
      if (r < 2 * my) {
        const int f = r / my;
        j = r - f * my;
        i = f == 0 ? 0 : mx - 1;
      } else {
        const int r2 = r - 2 * my, f = r2 / mx;
        i = r2 - f * mx;
        j = f == 0 ? 0 : my - 1;
      }
      cp_async8(RZ + r, e + (h.ox + i) + (h.oy + j) * esy + (h.oz - 1) * esz);
    }
  stage_raw(0);
  stage_raw(1);
#ifdef ASDSM_H3_TRACE
  long long ph[4] = {0, 0, 0, 0}, c0 = clock64(), c1, c2, c3, c4;
#endif
  // pair sums of chunk ci from its staged raw ring values: (plane, sign) -> y transform of
  // cx0 A0 +/- cx1 A1, x transform of cy0 B0 +/- cy1 B1
  auto pairs_chunk = [&](int ci) {
    const int t0 = ci * TC;
    const int np = min(TC, mt - t0);
    const double* RW = RAW + (ci & 1) * TC * nring;
    fwd_pairs(Ty, 2 * np, [&](int v, int j) {
      const int tt = v >> 1;
      const double* rp = RW + tt * nring;
      const bool z0 = t0 + tt == 0;
      const double r0 = ring_raw(rp, RZ[j], 0, j, z0);
      const double r1 = mx > 1 ? ring_raw(rp, RZ[my + j], mx - 1, j, z0) : 0.0;
      const double a0 = cx0 * r0, a1 = cx1 * r1;
      return (v & 1) ? a0 - a1 : a0 + a1;
    }, HB);
    fwd_pairs(Tx, 2 * np, [&](int v, int i) {
      const int tt = v >> 1;
      const double* rp = RW + tt * nring;
      const bool z0 = t0 + tt == 0;
      const bool mid = i > 0 && i < mx - 1;
      const double r0 = mid ? ring_raw(rp, RZ[2 * my + i], i, 0, z0) : 0.0;
      const double r1 = (mid && my > 1) ? ring_raw(rp, RZ[2 * my + mx + i], i, my - 1, z0) : 0.0;
      const double b0 = cy0 * r0, b1 = cy1 * r1;
      return (v & 1) ? b0 - b1 : b0 + b1;
    }, HBx);
  };
  // Chunk schedule (4 CTA barriers per chunk): [top barrier] stage raw(ci+2), dots(ci) -> V |
  // line steps -> X | step A | step B, then -- with no barrier -- the pair sums of chunk ci+1:
  // they read RAW(ci+1) (landed before step A's barrier: the wait below) and write HB, which
  // the dots of chunk ci released two barriers ago, so they fill the tail of step B.
  asm volatile("cp.async.wait_group 1;\n" ::: "memory");
  __syncthreads();
  for (int t0 = -TC; t0 < mt; t0 += TC) {  // the first pass only forms the pair sums of chunk 0
    const int np = min(TC, mt - t0);
    const int ci = t0 / TC;
    if (t0 < 0) {
      pairs_chunk(0);
      continue;
    }
    __syncthreads();  // pair sums complete, RAW(ci) consumed, X free (step B of chunk ci-1 done)
    stage_raw(ci + 2);  // this chunk's raw values are consumed (pair sums formed)
    {  // both axes' dots as one task list over the warps (16 tiles at config 4: one per warp)
      const int nty_ = fwd_mma_tasks(Ty, 2 * np), ntx_ = fwd_mma_tasks(Tx, 2 * np);
      for (int task = tid >> 5; task < nty_ + ntx_; task += kH3Warps) {
        if (task < nty_)
          fwd_dots_mma(Ty, 2 * np, HB, task, [&](int v, int l, double x) { V[(v >> 1) * nring + (v & 1) * my + l] = x; });
        else
          fwd_dots_mma(Tx, 2 * np, HBx, task - nty_,
                       [&](int v, int k, double x) { V[(v >> 1) * nring + 2 * my + (v & 1) * mx + k] = x; });
      }
    }
    __syncthreads();
#ifdef ASDSM_H3_TRACE
    c1 = clock64();
    ph[0] += c1 - c0;
#endif
    if (nlines > 0) {
      double iv[NL], s0y[NL];  // bidiagonal: one pivot per line for every t (L1-resident table)
#pragma unroll
      for (int u = 0; u < NL; ++u) {
        const int l = tl0 + LG * u;
        iv[u] = u < nlines ? __ldg(A.ipiv + tk + mx * l) : 0.0;
        s0y[u] = u < nlines ? Ty.s0(l) : 0.0;
      }
      const double s0x = Tx.s0(tk);
      const int v1 = (tk & 1) * my + tl0, v2 = 2 * my + (tl0 & 1) * mx + tk;
      const int xo = rowof(tl0) * skx + Tx.col(tk), xs = (LG >> 1) * skx;
      for (int tt = 0; tt < np; ++tt) {
        const int t = t0 + tt;
        const double* Vp = V + tt * nring;
        double* Xp = X + tt * ps + xo;
        const double xb = Vp[v2];
#pragma unroll
        for (int u = 0; u < NL; ++u) {
          if (u >= nlines) break;
          double f = s0x * Vp[v1 + LG * u];
          f = fma(s0y[u], xb, f);
          if (t == 0) f += CH0[(tl0 + LG * u) * mx + tk];
          const double y = (t == 0) ? f * iv[u] : (f - lft * yv[u]) * iv[u];
          yv[u] = y;
          Xp[u * xs] = y;
        }
      }
    }
    __syncthreads();
    asm volatile("cp.async.wait_group 1;\n" ::: "memory");  // RAW(ci+1): visible after step A's barrier
#ifdef ASDSM_H3_TRACE
    c2 = clock64();
    back_planes(X, np, t0, Tx, Ty, A, h, e, &c3);
    c4 = clock64();
    if (t0 + TC < mt) pairs_chunk(ci + 1);
    ph[1] += c2 - c1;
    ph[2] += c3 - c2;
    ph[3] += c4 - c3;
    c0 = c4;
#else
    back_planes(X, np, t0, Tx, Ty, A, h, e);
    if (t0 + TC < mt) pairs_chunk(ci + 1);
#endif
  }
#ifdef ASDSM_H3_TRACE
  if (tid == 0 && (blockIdx.x == 0 || blockIdx.x == 500))
    printf("H3TRACE blk %d fwd %lld thomas %lld stepA %lld stepB %lld\n", blockIdx.x, ph[0], ph[1], ph[2], ph[3]);
#endif
}

int stride4mod8(int m) {  // >= round_up(m, 4) and == 4 (mod 8): conflict-free DMMA fragments
  int s = (m + 3) & ~3;
  if (s % 8 != 4) s += 4;
  return s;
}

H3Axis axis_of(int m) {
  H3Axis a{};
  a.m = m;
  a.he = (m + 1) / 2;
  a.ho = m / 2;
  a.khe = (a.he + 3) & ~3;
  a.kho = (a.ho + 3) & ~3;
  a.hrow = (a.he + 7) & ~7;
  a.sh = stride4mod8(a.khe + a.kho);
  return a;
}

}  // namespace

bool hole3d_fused_plan(Hole3DFusedArgs& A, bool causal) {
  const int mx = A.m[0], my = A.m[1], mt = A.m[2];
  if (mx < 1 || my < 1 || mt < 1 || mx > 64 || my > 64) return false;
  A.ax = axis_of(mx);
  A.ay = axis_of(my);
  H3Layout& L = A.lay;
  L.kxo = A.ax.kho;
  L.kyo = A.ay.kho;
  L.rp = A.ay.khe + A.ay.kho;                            // plane rows (even/odd l, zero gaps)
  L.skx = stride4mod8(std::max(A.ax.khe + A.ax.kho, mx));  // row: even/odd k, or natural i
  L.ntx = A.ax.hrow * A.ax.sh + 2 * mx;
  L.nty = A.ay.hrow * A.ay.sh + 2 * my;
  L.tx = 0;
  L.ty = (L.ntx + 1) & ~1;
  size_t off = L.ty + ((L.nty + 1) & ~1);
  const size_t kMax = 227 * 1024 / sizeof(double);
  const size_t slack = 8 * static_cast<size_t>(L.skx) + 8;
  if (!causal) {
    if (mx * my > kSymLines * kH3Threads) return false;
    L.tc = mt;
    L.faces = static_cast<int>(off);
    off += 2 * static_cast<size_t>(mt) * my + 2 * static_cast<size_t>(mt) * mx + 2 * static_cast<size_t>(my) * mx;
    off = (off + 1) & ~static_cast<size_t>(1);
    L.x = static_cast<int>(off);
    size_t xs = static_cast<size_t>(mt) * L.rp * L.skx + slack;
    // scratch: faces + pair sums (YA/XB batches), z face + G + pair sums
    xs = std::max(xs, 2 * static_cast<size_t>(mt) * (mx + my) + 4 * static_cast<size_t>(mt) * (A.ax.he + A.ay.he));
    xs = std::max(xs, 2 * static_cast<size_t>(mx) * my + 2 * static_cast<size_t>(std::max(mx, my)) * (A.ax.he + A.ay.he));
    L.xsize = static_cast<int>(xs);
    off += xs;
    if (off > kMax) return false;
  } else {
    if (mx * my > kCausalLines * kH3Threads) return false;
    // line ownership: thread (k, l0) takes l = l0 + lg u; lg even (one l parity per thread)
    L.lg = std::max(2, std::min(kH3Threads / mx, (my + 1) & ~1) & ~1);
    L.lu = (my + L.lg - 1) / L.lg;
    if (L.lu > kCausalLines || mx * std::min(L.lg, my) > kH3Threads) return false;
    const int nring = 2 * (mx + my);
    L.faces = static_cast<int>(off);
    int tc = 0;
    const int tc_max = std::getenv("ASDSM_H3_TC") ? std::atoi(std::getenv("ASDSM_H3_TC")) : 8;
    // Among the chunk sizes that fit, the one with the least modelled time: per chunk the
    // step-A rounds (8-row blocks over 16 warps), the step-B rounds ((plane, j tile, n quad)
    // tasks over 16 warps) and a fixed per-chunk cost (ring transforms, barriers), in the
    // proportions measured at config 4 (clock64 trace of the round-2 kernel: 5.0 / 6.4 k cycles
    // per round, 4.9 k per chunk; the line steps cost per plane, not per chunk).
    const int nty = (A.ay.he + 7) / 8, nq = ((mx + 7) / 8 + 3) / 4;
    double best = 1e300;
    for (int c = std::min(mt, tc_max); c >= 1; --c) {
      size_t o = off + static_cast<size_t>(my) * mx + 3 * static_cast<size_t>(c) * nring + nring +
                 4 * static_cast<size_t>(c) * (A.ax.he + A.ay.he);
      o = (o + 1) & ~static_cast<size_t>(1);
      size_t xs = static_cast<size_t>(c) * L.rp * L.skx + slack;
      xs = std::max(xs, 2 * static_cast<size_t>(mx) * my + 2 * static_cast<size_t>(std::max(mx, my)) * (A.ax.he + A.ay.he));
      if (o + xs > kMax) continue;
      const int ra = (c * L.rp + 7) / 8, rb = c * nty * nq;
      const double t = ((mt + c - 1) / c) * (5.0 * ((ra + kH3Warps - 1) / kH3Warps) + 6.4 * ((rb + kH3Warps - 1) / kH3Warps) + 4.9);
      if (t < best) {
        best = t;
        tc = c;
      }
    }
    if (tc == 0) return false;
    L.tc = tc;
    off += static_cast<size_t>(my) * mx + 3 * static_cast<size_t>(tc) * nring + nring +
           4 * static_cast<size_t>(tc) * (A.ax.he + A.ay.he);
    off = (off + 1) & ~static_cast<size_t>(1);
    L.x = static_cast<int>(off);
    size_t xs = static_cast<size_t>(tc) * L.rp * L.skx + slack;
    xs = std::max(xs, 2 * static_cast<size_t>(mx) * my + 2 * static_cast<size_t>(std::max(mx, my)) * (A.ax.he + A.ay.he));
    L.xsize = static_cast<int>(xs);
    off += xs;
  }
  L.bytes = off * sizeof(double);
  return true;
}

std::vector<double> hole3d_half_table(const H3Axis& a, const std::vector<double>& half) {
  // half: SepSolver::half layout [half_sine_rows][2 kh] (col k/2 | kh + k/2), then sc[m], ci[m]
  const int m = a.m, kh = half_sine_kh(m), hr = half_sine_rows(m);
  std::vector<double> t(static_cast<size_t>(a.hrow) * a.sh + 2 * static_cast<size_t>(m), 0.0);
  for (int i = 0; i < a.he; ++i)
    for (int k = 0; k < m; ++k) {
      const int src = (k & 1) ? kh + (k >> 1) : (k >> 1);
      const int dst = (k & 1) ? a.khe + (k >> 1) : (k >> 1);
      t[static_cast<size_t>(i) * a.sh + dst] = half[static_cast<size_t>(i) * 2 * kh + src];
    }
  for (int i = 0; i < 2 * m; ++i)
    t[static_cast<size_t>(a.hrow) * a.sh + i] = half[static_cast<size_t>(hr) * 2 * kh + i];
  return t;
}

void launch_hole3d_fused(double* e, const Hole3DFusedArgs& A, bool causal, DevState* st, cudaStream_t s) {
  const unsigned nh = static_cast<unsigned>(A.nbox[0] * A.nbox[1] * A.nbox[2]);
  if (causal && A.lay.lu <= 5) hole3d_fused_kernel<true, 5><<<nh, kH3Threads, A.lay.bytes, s>>>(e, A, st);
  else if (causal) hole3d_fused_kernel<true><<<nh, kH3Threads, A.lay.bytes, s>>>(e, A, st);
  else hole3d_fused_kernel<false><<<nh, kH3Threads, A.lay.bytes, s>>>(e, A, st);
  ASDSM_CUDA_CHECK(cudaGetLastError());
  ++g_kernel_launches;
}

void hole3d_fused_prepare() {  // outside any stream capture: the dynamic shared-memory limit
  static bool done = false;
  if (done) return;
  done = true;
  const int mx = 227 * 1024;
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole3d_fused_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole3d_fused_kernel<true, 5>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
  ASDSM_CUDA_CHECK(cudaFuncSetAttribute(hole3d_fused_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
}

}  // namespace asdsm_b200
