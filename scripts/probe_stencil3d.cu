// Probe: shapes of the 3D fine-grid residual pass r = b - A u (7-point stencil, x fastest, odd
// row lengths) on one B200 -- which tile shape / walk order streams closest to the HBM copy rate.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o probe_stencil3d probe_stencil3d.cu
//   ./probe_stencil3d N [exact]      (N = 509 or 259)
// Every variant computes the same non-contracted row sum (z-, y-, x-, c, x+, y+, z+), so the
// checksums must agree bitwise.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

typedef long long i64;
struct St { double l[3], d, r[3]; };
struct Args {
  const double* u; const double* b; const double* ex; double* r; double* part;
  int Nx, Ny, Nz; i64 sy, sz, n; St st;
};

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("cuda error %s at %d\n", cudaGetErrorString(e_), __LINE__); exit(1); } } while (0)

__device__ __forceinline__ double row_sum(const St& st, bool zl, bool yl, bool xl, bool xr, bool yr, bool zr,
                                          double vzl, double vyl, double vxl, double vc, double vxr, double vyr, double vzr) {
  double acc = 0.0;
  if (zl) acc = __dadd_rn(acc, __dmul_rn(st.l[2], vzl));
  if (yl) acc = __dadd_rn(acc, __dmul_rn(st.l[1], vyl));
  if (xl) acc = __dadd_rn(acc, __dmul_rn(st.l[0], vxl));
  acc = __dadd_rn(acc, __dmul_rn(st.d, vc));
  if (xr) acc = __dadd_rn(acc, __dmul_rn(st.r[0], vxr));
  if (yr) acc = __dadd_rn(acc, __dmul_rn(st.r[1], vyr));
  if (zr) acc = __dadd_rn(acc, __dmul_rn(st.r[2], vzr));
  return acc;
}

__device__ __forceinline__ void block_fold(double a0, double a1, double a2, double a3, double* part) {
  __shared__ double sh[4][32];
  for (int o = 16; o; o >>= 1) {
    a0 += __shfl_xor_sync(~0u, a0, o);
    a1 = fmax(a1, __shfl_xor_sync(~0u, a1, o));
    a2 += __shfl_xor_sync(~0u, a2, o);
    a3 = fmax(a3, __shfl_xor_sync(~0u, a3, o));
  }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = (blockDim.x + 31) >> 5;
  if (l == 0) { sh[0][w] = a0; sh[1][w] = a1; sh[2][w] = a2; sh[3][w] = a3; }
  __syncthreads();
  if (w == 0) {
    a0 = l < nw ? sh[0][l] : 0.0; a1 = l < nw ? sh[1][l] : 0.0; a2 = l < nw ? sh[2][l] : 0.0; a3 = l < nw ? sh[3][l] : 0.0;
    for (int o = 16; o; o >>= 1) {
      a0 += __shfl_xor_sync(~0u, a0, o);
      a1 = fmax(a1, __shfl_xor_sync(~0u, a1, o));
      a2 += __shfl_xor_sync(~0u, a2, o);
      a3 = fmax(a3, __shfl_xor_sync(~0u, a3, o));
    }
    if (l == 0) {
      double* p = part + 4 * blockIdx.x;
      p[0] = a0; p[1] = a1; p[2] = a2; p[3] = a3;
    }
  }
}

// ---- copy-rate calibrations: r = b - d u, linear vs (TX x TY x ZC) tiles
__global__ void __launch_bounds__(256) lin_copy(Args A) {
  const i64 n2 = A.n / 2, stride = (i64)gridDim.x * blockDim.x;
  for (i64 i = (i64)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    const double2 u = __ldg((const double2*)A.u + i), b = __ldg((const double2*)A.b + i);
    ((double2*)A.r)[i] = make_double2(b.x - A.st.d * u.x, b.y - A.st.d * u.y);
  }
}
template <int TXW, int TYH, int ZCN>
__global__ void __launch_bounds__(256) tile_copy(Args A) {
  const int ntx = (A.Nx + TXW - 1) / TXW, nty = (A.Ny + TYH - 1) / TYH, ntz = (A.Nz + ZCN - 1) / ZCN;
  const i64 ntiles = (i64)ntx * nty * ntz;
  const int tx = threadIdx.x % TXW, ty = threadIdx.x / TXW;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int bx = t % ntx, by = (t / ntx) % nty, bz = t / ((i64)ntx * nty);
    const int x = bx * TXW + tx, y = by * TYH + ty;
    if (x >= A.Nx || y >= A.Ny) continue;
#pragma unroll
    for (int q = 0; q < ZCN; ++q) {
      const int z = bz * ZCN + q;
      if (z >= A.Nz) break;
      const i64 p = x + y * A.sy + z * A.sz;
      A.r[p] = __ldg(A.b + p) - A.st.d * __ldg(A.u + p);
    }
  }
}

// ---- V_zc: the current kernel's shape generalised: persistent CTAs over (TXW x TYH x ZCN) tiles,
// TXW*TYH = 256 threads, z neighbours in registers, x/y neighbours through L1
template <int TXW, int TYH, int ZCN, bool EX, int MINB>
__global__ void __launch_bounds__(256, MINB) zc_kernel(Args A) {
  const int Nx = A.Nx, Ny = A.Ny, Nz = A.Nz;
  const i64 sy = A.sy, sz = A.sz;
  const St& st = A.st;
  const double* __restrict__ uu = A.u;
  const int ntx = (Nx + TXW - 1) / TXW, nty = (Ny + TYH - 1) / TYH, ntz = (Nz + ZCN - 1) / ZCN;
  const i64 ntiles = (i64)ntx * nty * ntz;
  const int tx = threadIdx.x % TXW, ty = threadIdx.x / TXW;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int bx = t % ntx, by = (t / ntx) % nty, bz = t / ((i64)ntx * nty);
    const int x = bx * TXW + tx, y = by * TYH + ty, z0 = bz * ZCN;
    if (x >= Nx || y >= Ny) continue;
    const i64 pxy = x + y * sy;
    double vz[ZCN + 2];
#pragma unroll
    for (int q = 0; q < ZCN + 2; ++q) {
      const int z = z0 - 1 + q;
      vz[q] = (z >= 0 && z < Nz) ? __ldg(uu + pxy + z * sz) : 0.0;
    }
#pragma unroll
    for (int q = 0; q < ZCN; ++q) {
      const int z = z0 + q;
      if (z >= Nz) break;
      const i64 p = pxy + z * sz;
      const double vc = vz[q + 1];
      const double acc = row_sum(st, z > 0, y > 0, x > 0, x < Nx - 1, y < Ny - 1, z < Nz - 1, vz[q],
                                 y > 0 ? __ldg(uu + p - sy) : 0.0, x > 0 ? __ldg(uu + p - 1) : 0.0, vc,
                                 x < Nx - 1 ? __ldg(uu + p + 1) : 0.0, y < Ny - 1 ? __ldg(uu + p + sy) : 0.0, vz[q + 2]);
      const double r = __dsub_rn(__ldg(A.b + p), acc);
      A.r[p] = r;
      a0 += r * r; a1 = fmax(a1, fabs(r));
      if (EX) { const double d = vc - __ldg(A.ex + p); a2 += d * d; a3 = fmax(a3, fabs(d)); }
    }
  }
  block_fold(a0, a1, a2, a3, A.part);
}

// ---- V_lin: the array as one linear stream; thread-per-point, P points per thread a block
// stride apart (coalesced), neighbours p+-1, p+-Nx, p+-NxNy through L1/L2; blocks in linear order
template <int P, bool EX, int MINB>
__global__ void __launch_bounds__(256, MINB) lin_kernel(Args A) {
  const int Nx = A.Nx, Ny = A.Ny, Nz = A.Nz;
  const i64 sy = A.sy, sz = A.sz, n = A.n;
  const St& st = A.st;
  const double* __restrict__ uu = A.u;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  const i64 chunk = 256 * P;
  for (i64 base = (i64)blockIdx.x * chunk; base < n; base += (i64)gridDim.x * chunk) {
    double vc[P], vxl[P], vxr[P], vyl[P], vyr[P], vzl[P], vzr[P], bb[P], ee[P];
    int xs[P], ys[P], zs[P];
#pragma unroll
    for (int k = 0; k < P; ++k) {
      const i64 p = base + k * 256 + threadIdx.x;
      const bool in = p < n;
      const int z = (int)(p / sz);
      const int rem = (int)(p - (i64)z * sz);
      const int y = rem / Nx, x = rem - y * Nx;
      xs[k] = in ? x : -1; ys[k] = y; zs[k] = z;
      vc[k] = in ? __ldg(uu + p) : 0.0;
      vxl[k] = (in && x > 0) ? __ldg(uu + p - 1) : 0.0;
      vxr[k] = (in && x < Nx - 1) ? __ldg(uu + p + 1) : 0.0;
      vyl[k] = (in && y > 0) ? __ldg(uu + p - sy) : 0.0;
      vyr[k] = (in && y < Ny - 1) ? __ldg(uu + p + sy) : 0.0;
      vzl[k] = (in && z > 0) ? __ldg(uu + p - sz) : 0.0;
      vzr[k] = (in && z < Nz - 1) ? __ldg(uu + p + sz) : 0.0;
      bb[k] = in ? __ldg(A.b + p) : 0.0;
      if (EX) ee[k] = in ? __ldg(A.ex + p) : 0.0;
    }
#pragma unroll
    for (int k = 0; k < P; ++k) {
      if (xs[k] < 0) continue;
      const i64 p = base + k * 256 + threadIdx.x;
      const int x = xs[k], y = ys[k], z = zs[k];
      const double acc = row_sum(st, z > 0, y > 0, x > 0, x < Nx - 1, y < Ny - 1, z < Nz - 1, vzl[k], vyl[k], vxl[k],
                                 vc[k], vxr[k], vyr[k], vzr[k]);
      const double r = __dsub_rn(bb[k], acc);
      A.r[p] = r;
      a0 += r * r; a1 = fmax(a1, fabs(r));
      if (EX) { const double d = vc[k] - ee[k]; a2 += d * d; a3 = fmax(a3, fabs(d)); }
    }
  }
  block_fold(a0, a1, a2, a3, A.part);
}

// ---- V_slab: a CTA owns RY consecutive full rows (RY*Nx contiguous points of one plane) and
// ZCN planes: thread t takes the in-slab linear offsets t, t+256, ... ; z neighbours in
// registers, y neighbours within the slab come from the same CTA's L1 lines
template <int RY, int ZCN, bool EX, int MINB>
__global__ void __launch_bounds__(256, MINB) slab_kernel(Args A) {
  const int Nx = A.Nx, Ny = A.Ny, Nz = A.Nz;
  const i64 sy = A.sy, sz = A.sz;
  const St& st = A.st;
  const double* __restrict__ uu = A.u;
  const int nty = (Ny + RY - 1) / RY, ntz = (Nz + ZCN - 1) / ZCN;
  const i64 ntiles = (i64)nty * ntz;
  double a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  for (i64 t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int by = t % nty, bz = t / nty;
    const int y0 = by * RY, z0 = bz * ZCN;
    const int rows = min(RY, Ny - y0);
    const int npts = rows * Nx;
    for (int o = threadIdx.x; o < npts; o += 256) {
      const int yy = o / Nx, x = o - yy * Nx, y = y0 + yy;
      const i64 pxy = x + y * sy;
      double vz[ZCN + 2];
#pragma unroll
      for (int q = 0; q < ZCN + 2; ++q) {
        const int z = z0 - 1 + q;
        vz[q] = (z >= 0 && z < Nz) ? __ldg(uu + pxy + z * sz) : 0.0;
      }
#pragma unroll
      for (int q = 0; q < ZCN; ++q) {
        const int z = z0 + q;
        if (z >= Nz) break;
        const i64 p = pxy + z * sz;
        const double vc = vz[q + 1];
        const double acc = row_sum(st, z > 0, y > 0, x > 0, x < Nx - 1, y < Ny - 1, z < Nz - 1, vz[q],
                                   y > 0 ? __ldg(uu + p - sy) : 0.0, x > 0 ? __ldg(uu + p - 1) : 0.0, vc,
                                   x < Nx - 1 ? __ldg(uu + p + 1) : 0.0, y < Ny - 1 ? __ldg(uu + p + sy) : 0.0, vz[q + 2]);
        const double r = __dsub_rn(__ldg(A.b + p), acc);
        A.r[p] = r;
        a0 += r * r; a1 = fmax(a1, fabs(r));
        if (EX) { const double d = vc - __ldg(A.ex + p); a2 += d * d; a3 = fmax(a3, fabs(d)); }
      }
    }
  }
  block_fold(a0, a1, a2, a3, A.part);
}

static double checksum(const double* d_r, i64 n) {
  std::vector<double> h(n);
  CK(cudaMemcpy(h.data(), d_r, n * 8, cudaMemcpyDeviceToHost));
  unsigned long long s = 0;
  for (i64 i = 0; i < n; ++i) { unsigned long long v; memcpy(&v, &h[i], 8); s = s * 1000003ull + v; }
  return (double)(s % 1000000007ull);
}

template <typename F>
static void run(const char* name, F launch, Args& A, double bytes, float* flush, size_t flush_n, bool check = true) {
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaMemset(A.r, 0, A.n * 8));
  float best = 1e30f, sum = 0;
  const int reps = 6;
  for (int i = 0; i < reps + 2; ++i) {
    CK(cudaMemsetAsync(flush, i, flush_n));
    CK(cudaEventRecord(e0));
    launch();
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    CK(cudaGetLastError());
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    if (i >= 2) { best = ms < best ? ms : best; sum += ms; }
  }
  const double cs = check ? checksum(A.r, A.n) : 0.0;
  printf("%-34s mean %8.4f ms  best %8.4f ms  %7.1f GB/s (mean)  %7.1f (best)  checksum %.0f\n", name, sum / reps, best,
         bytes / (sum / reps) / 1e6, bytes / best / 1e6, cs);
  fflush(stdout);
}

int main(int argc, char** argv) {
  const int N = argc > 1 ? atoi(argv[1]) : 509;
  const bool ex = argc > 2 && atoi(argv[2]);
  Args A{};
  A.Nx = A.Ny = A.Nz = N; A.sy = N; A.sz = (i64)N * N; A.n = (i64)N * N * N;
  const double h = 1.0 / (N + 1);
  for (int a = 0; a < 3; ++a) { A.st.l[a] = -1.0 / (h * h) - 0.5 / (2 * h); A.st.r[a] = -1.0 / (h * h) + 0.5 / (2 * h); }
  A.st.d = 6.0 / (h * h);
  double *u, *b, *x, *r, *part;
  CK(cudaMalloc(&u, (A.n + 2) * 8)); CK(cudaMalloc(&b, (A.n + 2) * 8)); CK(cudaMalloc(&x, (A.n + 2) * 8));
  CK(cudaMalloc(&r, (A.n + 2) * 8)); CK(cudaMalloc(&part, 4 * 65536 * 8));
  {
    std::vector<double> h0(A.n);
    unsigned long long s = 88172645463325252ull;
    auto rnd = [&]() { s ^= s << 13; s ^= s >> 7; s ^= s << 17; return (double)(s >> 11) / 9007199254740992.0 - 0.5; };
    for (auto& v : h0) v = rnd();
    CK(cudaMemcpy(u, h0.data(), A.n * 8, cudaMemcpyHostToDevice));
    for (auto& v : h0) v = rnd();
    CK(cudaMemcpy(b, h0.data(), A.n * 8, cudaMemcpyHostToDevice));
    for (auto& v : h0) v = rnd();
    CK(cudaMemcpy(x, h0.data(), A.n * 8, cudaMemcpyHostToDevice));
  }
  A.u = u; A.b = b; A.ex = x; A.r = r; A.part = part;
  const size_t flush_n = 512u << 20;
  float* flush; CK(cudaMalloc(&flush, flush_n));
  const double by = (ex ? 32.0 : 24.0) * A.n, by_copy = 24.0 * A.n;
  const int SM = 148;
  printf("N = %d, exact = %d, %.1f M points, algorithmic %.2f GB\n", N, (int)ex, A.n / 1e6, by / 1e9);
  run("lin_copy (8x148)", [&] { lin_copy<<<8 * SM, 256>>>(A); }, A, by_copy, flush, flush_n, false);
  run("lin_copy (32x148)", [&] { lin_copy<<<32 * SM, 256>>>(A); }, A, by_copy, flush, flush_n, false);
  run("tile_copy 32x8x8", [&] { tile_copy<32, 8, 8><<<8 * SM, 256>>>(A); }, A, by_copy, flush, flush_n, false);
  run("tile_copy 64x4x8", [&] { tile_copy<64, 4, 8><<<8 * SM, 256>>>(A); }, A, by_copy, flush, flush_n, false);
  run("tile_copy 128x2x8", [&] { tile_copy<128, 2, 8><<<8 * SM, 256>>>(A); }, A, by_copy, flush, flush_n, false);
  run("tile_copy 256x1x8", [&] { tile_copy<256, 1, 8><<<8 * SM, 256>>>(A); }, A, by_copy, flush, flush_n, false);
  run("tile_copy 32x8x1", [&] { tile_copy<32, 8, 1><<<8 * SM, 256>>>(A); }, A, by_copy, flush, flush_n, false);
#define ZCV(TX, TY, ZC, MB, G)                                                                                     \
  if (ex) run("zc " #TX "x" #TY "x" #ZC " minb" #MB " grid" #G, [&] { zc_kernel<TX, TY, ZC, true, MB><<<G * SM, 256>>>(A); }, A, by, flush, flush_n); \
  else run("zc " #TX "x" #TY "x" #ZC " minb" #MB " grid" #G, [&] { zc_kernel<TX, TY, ZC, false, MB><<<G * SM, 256>>>(A); }, A, by, flush, flush_n);
  ZCV(32, 8, 8, 4, 8)
  ZCV(32, 8, 8, 4, 4)
  ZCV(32, 8, 4, 4, 8)
  ZCV(32, 8, 4, 6, 6)
  ZCV(32, 8, 2, 8, 8)
  ZCV(64, 4, 8, 4, 8)
  ZCV(128, 2, 8, 4, 8)
  ZCV(256, 1, 8, 4, 8)
  ZCV(64, 4, 4, 6, 6)
  ZCV(128, 2, 4, 6, 6)
  ZCV(256, 1, 4, 6, 6)
#define LINV(P, MB, G)                                                                                             \
  if (ex) run("lin P" #P " minb" #MB " grid" #G, [&] { lin_kernel<P, true, MB><<<G, 256>>>(A); }, A, by, flush, flush_n); \
  else run("lin P" #P " minb" #MB " grid" #G, [&] { lin_kernel<P, false, MB><<<G, 256>>>(A); }, A, by, flush, flush_n);
  const int gfull1 = (int)((A.n + 255) / 256), gfull2 = (int)((A.n + 511) / 512), gfull4 = (int)((A.n + 1023) / 1024);
  LINV(1, 8, gfull1)
  LINV(2, 6, gfull2)
  LINV(4, 4, gfull4)
  LINV(1, 8, 8 * SM)
  LINV(2, 6, 6 * SM)
  LINV(4, 4, 4 * SM)
  LINV(2, 4, 8 * SM)
#define SLV(RY, ZC, MB, G)                                                                                         \
  if (ex) run("slab RY" #RY " ZC" #ZC " minb" #MB " grid" #G, [&] { slab_kernel<RY, ZC, true, MB><<<G * SM, 256>>>(A); }, A, by, flush, flush_n); \
  else run("slab RY" #RY " ZC" #ZC " minb" #MB " grid" #G, [&] { slab_kernel<RY, ZC, false, MB><<<G * SM, 256>>>(A); }, A, by, flush, flush_n);
  SLV(4, 4, 6, 6)
  SLV(8, 4, 6, 6)
  SLV(8, 8, 4, 8)
  SLV(16, 4, 6, 6)
  SLV(4, 2, 8, 8)
  SLV(8, 2, 8, 8)
  return 0;
}
