// Host-side plan for the B200 ASDSM solver: mesh geometry, stencil coefficients, the
// separable direct-solver tables for every box type (slabs, holes), and device buffers.
//
// Mirrors the reference's SolverContext (proj/include/asdsm/solver.hpp:114-155): everything
// the outer iteration reuses across steps is built once here and kept resident in HBM.
#pragma once
#include <array>
#include <complex>
#include <memory>
#include <string>
#include <vector>

#include "common.cuh"

namespace asdsm_b200 {

// Error codes mirror the reference's exception classes (proj/include/asdsm/errors.hpp:8-66).
enum ErrorCode {
  kOk = 0,
  kError = 1,
  kDivisibilityError = 2,
  kDegenerateError = 3,
  kIndexOutOfRange = 4,
  kNotASubmesh = 5,
  kInvalidKind = 6,
  kDimensionMismatch = 7,
  kSingularMatrix = 8,
  kSkeletonNotHollow = 9,
  kZeroNormSolution = 10,
  kUnknownExample = 11,
  kNoExactSolution = 12,
  kUnsupported = 13,
  kCudaFailure = 14,
};

struct AsdsmError : std::runtime_error {
  int code;
  AsdsmError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

// MeshConfig (proj/include/asdsm/mesh.hpp:56-83).
struct Mesh {
  int dim = 2;
  int nf[3] = {1, 1, 1};
  int nc[3] = {1, 1, 1};
  int n[3] = {1, 1, 1};      // refinement factors
  double h[3] = {0, 0, 0};   // fine steps
  double H[3] = {0, 0, 0};   // coarse steps
  int time_axis = -1;
  static Mesh create(int dim, const int* nf, const int* nc, int time_axis);
  int axis_points(unsigned mask, int a) const { return ((mask >> a) & 1u) ? nc[a] : nf[a]; }
  i64 point_count(unsigned mask) const;
  i64 hole_count() const;
};

// One tensor mesh kind (coarse mask) in its own x-fastest layout.
struct KindGeom {
  int dim = 2;
  int ext[3] = {1, 1, 1};
  i64 stride[3] = {0, 0, 0};
  i64 size = 0;
  unsigned mask = 0;
};
KindGeom kind_geom(const Mesh& m, unsigned mask);

// Per-axis 3-point stencil of the operator on one kind; reproduces fdm.cpp:63-82 exactly.
struct Stencil {
  int dim = 2;
  double left[3] = {0, 0, 0};
  double right[3] = {0, 0, 0};
  double dpart[3] = {0, 0, 0};  // this axis' diagonal contribution (2c or 1/h_t)
  int has_right[3] = {1, 1, 1};
  double diag = 0.0;            // accumulated 0.0 + dpart[0] + dpart[1] (+ dpart[2])
};
Stencil make_stencil(const Mesh& m, unsigned coarse_mask, const double* alpha, const double* beta);

// Where a batch of congruent boxes lives: element (box, idx) at
//   ptr + sum_a box_a * box_stride[a] + sum_a idx_a * stride[a]
struct BoxArray {
  double* ptr = nullptr;
  i64 stride[3] = {0, 0, 0};
  int nbox[3] = {1, 1, 1};
  i64 box_stride[3] = {0, 0, 0};
};

// Separable direct solver for A = sum_a I x..x T_a x..x I on one box type: every axis but the
// line axis L is diagonalized with the closed-form eigenvectors of the Toeplitz T_a, and
// the shifted 1D systems along L are solved by Thomas (many lines) or PCR (few long lines).
struct SepSolver {
  int dim = 2;
  int ext[3] = {1, 1, 1};
  int L = 0;
  int nd = 0;
  int dax[2] = {-1, -1};
  bool complex_modes = false;
  bool use_pcr = false;
  int ncombo = 1;
  double line_left = 0, line_right = 0;
  // device tables
  double* W[3] = {nullptr, nullptr, nullptr};  // forward V^{-1}: [k][j]
  double* V[3] = {nullptr, nullptr, nullptr};  // backward V: [j][k]
  double* Wt[3] = {nullptr, nullptr, nullptr}; // forward, transposed: [j][k] = W[k][j] (real only)
  // real only: even/odd half sine table [half_sine_rows][2 kh] (col(k) = k/2 | kh + (k-1)/2),
  // then scale_i [m] and (2/(m+1))/scale_i [m]  (plan.cpp half_sine_tables)
  double* half[3] = {nullptr, nullptr, nullptr};
  double* th_ipiv = nullptr;  // [pos][combo]
  double* th_cp = nullptr;    // [pos][combo]
  int pcr_levels = 0;
  double* pcr_k1 = nullptr;   // [combo][level][pos]
  double* pcr_k2 = nullptr;
  double* pcr_invb = nullptr; // [combo][pos]
  // Partition (separator) solve of one line by one warp (real modes, m <= kPartMaxLine): rows
  // q*M + M-1 (q < P-1, M = SEG + 1) are separators, lane q owns the SEG rows between
  // separators q-1 and q (the last lane m - (P-1) M <= SEG of them).  Per combo (stride
  // part_stride = 4 SEG + 352):
  //   [ipiv (SEG)] [g (SEG)] [h (SEG)] [g_last (SEG, zero padded)] [k1 (5 x 32)] [k2 (5 x 32)] [invb (32)]
  // ipiv: Thomas pivots of a segment; g/h: its responses to the left/right separator couplings;
  // k1/k2/invb: PCR of the reduced tridiagonal system over the P-1 separators.
  double* part = nullptr;
  int part_seg = 0, part_P = 0, part_last = 0, part_stride = 0;
  i64 mode_size() const { return static_cast<i64>(ext[0]) * ext[1] * (dim == 3 ? ext[2] : 1); }
};

// even/odd split sizes of an m-point sine transform: kh = padded half width (multiple of 4),
// rows = ceil(m/2) padded to a multiple of 8 (DMMA tile rows)
__host__ __device__ inline int half_sine_kh(int m) { return (((m + 1) / 2) + 3) & ~3; }
__host__ __device__ inline int half_sine_rows(int m) { return (((m + 1) / 2) + 7) & ~7; }

constexpr int kPartMaxSeg = 32;                         // rows per lane (registers)
constexpr int kPartMaxLine = 32 * (kPartMaxSeg + 1) - 2; // longest line the warp solve handles
__host__ __device__ inline int part_off_g(int seg) { return seg; }
__host__ __device__ inline int part_off_h(int seg) { return 2 * seg; }
__host__ __device__ inline int part_off_gl(int seg) { return 3 * seg; }
__host__ __device__ inline int part_off_k1(int seg) { return 4 * seg; }
__host__ __device__ inline int part_off_k2(int seg) { return 4 * seg + 160; }
__host__ __device__ inline int part_off_ib(int seg) { return 4 * seg + 320; }
__host__ __device__ inline int part_stride(int seg) { return 4 * seg + 352; }

struct DeviceAlloc {
  std::vector<void*> ptrs;
  template <typename T>
  T* alloc(size_t count) {
    void* p = nullptr;
    ASDSM_CUDA_CHECK(cudaMalloc(&p, count * sizeof(T) + 16));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
  void release_all();  // frees every allocation made so far
  ~DeviceAlloc();
};

// Build a separable solver (host tables in long double, uploaded once).
// `time_axis_in_box` marks an axis with the backward two-point stencil (not diagonalizable).
// `part_lines`: also build the warp-partition tables (SepSolver::part) when the lines are solved
// by per-thread Thomas (the 2D large-hole path solves them one warp per line instead).
SepSolver build_sep_solver(DeviceAlloc& dev, int dim, const int* ext, const Stencil& st,
                           int time_axis_in_box, int prefer_line_axis, i64 nbatch, const std::string& what,
                           bool part_lines = false);

}  // namespace asdsm_b200
