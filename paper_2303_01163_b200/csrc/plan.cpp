// Host-side plan construction: mesh validation, stencils, separable-solver tables.
#include "plan.hpp"

#include <algorithm>
#include <cmath>
#include <complex>

namespace asdsm_b200 {

using ld = long double;
using cld = std::complex<long double>;

void DeviceAlloc::release_all() {
  for (void* p : ptrs) cudaFree(p);
  ptrs.clear();
}

DeviceAlloc::~DeviceAlloc() { release_all(); }

// MeshConfig::create (proj/src/mesh.cpp:47-76): same validation order and messages.
Mesh Mesh::create(int dim, const int* nf, const int* nc, int time_axis) {
  if (dim < 2 || dim > 3)
    throw AsdsmError(kDimensionMismatch, "mesh dimension must be 2 or 3, got " + std::to_string(dim));
  if (time_axis != -1 && time_axis != dim - 1)
    throw AsdsmError(kDimensionMismatch, "time axis must be the last axis");
  Mesh m;
  m.dim = dim;
  m.time_axis = time_axis;
  for (int a = 0; a < dim; ++a) {
    const int f = nf[a], c = nc[a];
    if (f < 1 || c < 1)
      throw AsdsmError(kDegenerateError, "axis " + std::to_string(a) + ": interior point counts must be >= 1");
    if ((f + 1) % (c + 1) != 0)
      throw AsdsmError(kDivisibilityError, "axis " + std::to_string(a) + ": fine intervals " +
                                               std::to_string(f + 1) + " not divisible by coarse intervals " +
                                               std::to_string(c + 1));
    const int n = (f + 1) / (c + 1);
    if (n < 2)
      throw AsdsmError(kDegenerateError, "axis " + std::to_string(a) + ": refinement factor 1 leaves no holes");
    m.nf[a] = f;
    m.nc[a] = c;
    m.n[a] = n;
    m.h[a] = 1.0 / static_cast<double>(f + 1);
    m.H[a] = static_cast<double>(n) * m.h[a];
  }
  return m;
}

i64 Mesh::point_count(unsigned mask) const {
  i64 p = 1;
  for (int a = 0; a < dim; ++a) p *= axis_points(mask, a);
  return p;
}

i64 Mesh::hole_count() const {  // mesh.cpp:89-94
  i64 p = 1;
  for (int a = 0; a < dim; ++a) p *= static_cast<i64>(nc[a] + 1) * (n[a] - 1);
  return p;
}

KindGeom kind_geom(const Mesh& m, unsigned mask) {
  KindGeom g;
  g.dim = m.dim;
  g.mask = mask;
  i64 s = 1;
  for (int a = 0; a < 3; ++a) {
    g.ext[a] = a < m.dim ? m.axis_points(mask, a) : 1;
    g.stride[a] = s;
    s *= g.ext[a];
  }
  g.size = s;
  return g;
}

// axes_for_kind + axis_coeffs (proj/src/fdm.cpp:19-31, 63-82), constant coefficients.
Stencil make_stencil(const Mesh& m, unsigned coarse_mask, const double* alpha, const double* beta) {
  Stencil s;
  s.dim = m.dim;
  double diag = 0.0;
  for (int a = 0; a < m.dim; ++a) {
    const bool coarse = (coarse_mask >> a) & 1u;
    const double step = coarse ? m.H[a] : m.h[a];
    if (a == m.time_axis) {
      const double tc = 1.0 / step;
      diag += tc;
      s.dpart[a] = tc;
      s.left[a] = -tc;
      s.right[a] = 0.0;
      s.has_right[a] = 0;
      continue;
    }
    if (!(alpha[a] > 0.0))
      throw AsdsmError(kError, "diffusion coefficient not positive on axis " + std::to_string(a));
    const double c = alpha[a] / (step * step);
    const double d = beta[a] / (2.0 * step);
    diag += 2.0 * c;
    s.dpart[a] = 2.0 * c;
    s.left[a] = -c - d;
    s.right[a] = -c + d;
    s.has_right[a] = 1;
  }
  s.diag = diag;
  return s;
}

namespace {

template <typename T>
T* upload(DeviceAlloc& dev, const std::vector<T>& h) {
  T* d = dev.alloc<T>(h.size());
  ASDSM_CUDA_CHECK(cudaMemcpy(d, h.data(), h.size() * sizeof(T), cudaMemcpyHostToDevice));
  return d;
}

struct AxisEigen {
  bool cplx = false;
  std::vector<cld> lam;  // m
  std::vector<cld> V;    // [j][k]
  std::vector<cld> W;    // [k][j]
  std::vector<cld> scale;  // centred rho^j row scaling
  ld cond = 1;
};

// Closed-form eigenpairs of the Toeplitz tridiagonal T = tridiag(l, delta, r) of size m:
//   T v_k = lambda_k v_k,  v_k(j) = rho^j sin(j k pi/(m+1)),  rho = sqrt(l/r),
//   lambda_k = delta + 2 (l/rho) cos(k pi/(m+1)),  V^{-1} = 2/(m+1) S D^{-1}.
// The rho^j scaling is centred (rho^{j-(m+1)/2}) to balance magnitudes.
AxisEigen axis_eigen(int m, ld l, ld delta, ld r) {
  AxisEigen e;
  const cld q = cld(l / r, 0.0L);
  const cld rho = std::sqrt(q);
  e.cplx = (l / r) < 0.0L;
  const cld mu = cld(l, 0.0L) / rho;
  const ld pi = 3.141592653589793238462643383279502884L;
  const cld logrho = std::log(rho);
  e.lam.resize(static_cast<size_t>(m));
  for (int k = 0; k < m; ++k)
    e.lam[static_cast<size_t>(k)] = cld(delta, 0) + 2.0L * mu * std::cos(pi * static_cast<ld>(k + 1) / static_cast<ld>(m + 1));
  std::vector<cld> scale(static_cast<size_t>(m));
  ld smax = 0, smin = 1e300L;
  for (int j = 0; j < m; ++j) {
    const ld ex = static_cast<ld>(j + 1) - static_cast<ld>(m + 1) / 2.0L;
    scale[static_cast<size_t>(j)] = std::exp(ex * logrho);
    smax = std::max(smax, std::abs(scale[static_cast<size_t>(j)]));
    smin = std::min(smin, std::abs(scale[static_cast<size_t>(j)]));
  }
  e.cond = smax / smin;
  e.scale = scale;
  e.V.resize(static_cast<size_t>(m) * m);
  e.W.resize(static_cast<size_t>(m) * m);
  const i64 period = 2LL * (m + 1);
  for (int j = 0; j < m; ++j)
    for (int k = 0; k < m; ++k) {
      const i64 t = (static_cast<i64>(j + 1) * (k + 1)) % period;
      const ld s = std::sin(pi * static_cast<ld>(t) / static_cast<ld>(m + 1));
      e.V[static_cast<size_t>(j) * m + k] = scale[static_cast<size_t>(j)] * s;
      e.W[static_cast<size_t>(k) * m + j] = (2.0L / static_cast<ld>(m + 1)) * s / scale[static_cast<size_t>(j)];
    }
  return e;
}

// Thomas solve of tridiag(l, b, r) (size n) for rhs f, with the pivots ipiv (long double).
void thomas_ld(int n, ld l, ld r, const std::vector<ld>& ipiv, std::vector<ld>& x) {
  for (int t = 0; t < n; ++t) x[static_cast<size_t>(t)] = (t == 0 ? x[0] : x[static_cast<size_t>(t)] - l * x[static_cast<size_t>(t - 1)]) * ipiv[static_cast<size_t>(t)];
  for (int t = n - 2; t >= 0; --t) x[static_cast<size_t>(t)] -= r * ipiv[static_cast<size_t>(t)] * x[static_cast<size_t>(t + 1)];
}

// SepSolver::part tables (see plan.hpp): one warp solves a line of length m -- every lane a
// Thomas over its segment, a warp-PCR over the separators, then the segment reconstruction.
void build_partition_tables(SepSolver& s, int m, ld l, ld r, ld dL, const std::vector<cld>& sigma, DeviceAlloc& dev) {
  // segment lengths the device solve is instantiated for (slabstep2d.cu)
  static const int kSegs[] = {2, 4, 8, 12, 16, 20, 24, 28, 32};
  int SEG = 0, M = 0, P = 0, last = 0;
  for (int sg : kSegs) {
    M = sg + 1;
    P = (m + 1 + M - 1) / M;
    last = m - (P - 1) * M;
    if (P <= 32 && P >= 2 && last >= 1 && last <= sg) {
      SEG = sg;
      break;
    }
  }
  if (SEG == 0) return;
  const int R = P - 1;
  const int stride = part_stride(SEG);
  std::vector<double> tab(static_cast<size_t>(stride) * s.ncombo, 0.0);
  for (int c = 0; c < s.ncombo; ++c) {
    const ld b = dL + sigma[static_cast<size_t>(c)].real();
    std::vector<ld> ipiv(static_cast<size_t>(SEG));
    ld prev_cp = 0;
    for (int t = 0; t < SEG; ++t) {
      const ld w = t == 0 ? b : b - l * prev_cp;
      if (w == 0) throw AsdsmError(kSingularMatrix, "zero pivot in a partitioned line solve");
      ipiv[static_cast<size_t>(t)] = 1.0L / w;
      prev_cp = r * ipiv[static_cast<size_t>(t)];
    }
    std::vector<ld> g(static_cast<size_t>(M - 1), 0.0L), h(static_cast<size_t>(M - 1), 0.0L), gl(static_cast<size_t>(last), 0.0L);
    g[0] = l;
    thomas_ld(M - 1, l, r, ipiv, g);
    h[static_cast<size_t>(M - 2)] = r;
    thomas_ld(M - 1, l, r, ipiv, h);
    gl[0] = l;
    thomas_ld(last, l, r, ipiv, gl);
    // reduced system over the separators q < R
    std::vector<ld> A(static_cast<size_t>(std::max(R, 1)), 0.0L), B(A.size(), 0.0L), C(A.size(), 0.0L);
    for (int q = 0; q < R; ++q) {
      const bool next_full = q + 1 < P - 1;
      A[static_cast<size_t>(q)] = q >= 1 ? -l * g[static_cast<size_t>(M - 2)] : 0.0L;
      B[static_cast<size_t>(q)] = b - l * h[static_cast<size_t>(M - 2)] - r * (next_full ? g[0] : gl[0]);
      C[static_cast<size_t>(q)] = next_full ? -r * h[0] : 0.0L;
    }
    double* T = tab.data() + static_cast<size_t>(c) * stride;
    for (int t = 0; t < SEG; ++t) {
      T[t] = static_cast<double>(ipiv[static_cast<size_t>(t)]);
      T[part_off_g(SEG) + t] = static_cast<double>(g[static_cast<size_t>(t)]);
      T[part_off_h(SEG) + t] = static_cast<double>(h[static_cast<size_t>(t)]);
      if (t < last) T[part_off_gl(SEG) + t] = static_cast<double>(gl[static_cast<size_t>(t)]);
    }
    for (int lev = 0, stp = 1; lev < 5; ++lev, stp <<= 1) {
      std::vector<ld> A2(A.size()), B2(B.size()), C2(C.size());
      for (int i = 0; i < R; ++i) {
        ld f1 = 0, f2 = 0;
        const bool lo = i - stp >= 0, hi = i + stp < R;
        if (lo) f1 = A[static_cast<size_t>(i)] / B[static_cast<size_t>(i - stp)];
        if (hi) f2 = C[static_cast<size_t>(i)] / B[static_cast<size_t>(i + stp)];
        A2[static_cast<size_t>(i)] = lo ? -A[static_cast<size_t>(i - stp)] * f1 : 0.0L;
        C2[static_cast<size_t>(i)] = hi ? -C[static_cast<size_t>(i + stp)] * f2 : 0.0L;
        B2[static_cast<size_t>(i)] = B[static_cast<size_t>(i)] - (lo ? C[static_cast<size_t>(i - stp)] * f1 : 0.0L) -
                                    (hi ? A[static_cast<size_t>(i + stp)] * f2 : 0.0L);
        T[part_off_k1(SEG) + lev * 32 + i] = static_cast<double>(f1);
        T[part_off_k2(SEG) + lev * 32 + i] = static_cast<double>(f2);
      }
      A.swap(A2);
      B.swap(B2);
      C.swap(C2);
    }
    for (int i = 0; i < R; ++i) {
      if (B[static_cast<size_t>(i)] == 0) throw AsdsmError(kSingularMatrix, "zero pivot in a separator solve");
      T[part_off_ib(SEG) + i] = static_cast<double>(1.0L / B[static_cast<size_t>(i)]);
    }
  }
  s.part = upload(dev, tab);
  s.part_seg = SEG;
  s.part_P = P;
  s.part_last = last;
  s.part_stride = stride;
}

// Even/odd half of the sine factor of V = D S (plan.hpp SepSolver::half): rows i < ceil(m/2),
// column col(k) = k/2 (k even) or kh + (k-1)/2 (k odd), zero padded; then scale_i and
// (2/(m+1))/scale_i.  Row m-1-i of S is (-1)^k times row i, so a back transform needs only
// these rows: out(i) = scale_i (E_i + O_i), out(m-1-i) = scale_{m-1-i} (E_i - O_i).
std::vector<double> half_sine_tables(int m, const AxisEigen& e) {
  const int kh = half_sine_kh(m), rows = half_sine_rows(m);
  std::vector<double> t(static_cast<size_t>(rows) * 2 * kh + 2 * static_cast<size_t>(m), 0.0);
  const ld pi = 3.141592653589793238462643383279502884L;
  const i64 period = 2LL * (m + 1);
  for (int i = 0; i < (m + 1) / 2; ++i)
    for (int k = 0; k < m; ++k) {
      const i64 q = (static_cast<i64>(i + 1) * (k + 1)) % period;
      const int col = (k & 1) ? kh + (k >> 1) : (k >> 1);
      t[static_cast<size_t>(i) * 2 * kh + col] = static_cast<double>(std::sin(pi * static_cast<ld>(q) / static_cast<ld>(m + 1)));
    }
  double* sc = t.data() + static_cast<size_t>(rows) * 2 * kh;
  for (int i = 0; i < m; ++i) {
    const ld s = e.scale[static_cast<size_t>(i)].real();
    sc[i] = static_cast<double>(s);
    sc[m + i] = static_cast<double>((2.0L / static_cast<ld>(m + 1)) / s);
  }
  return t;
}

std::vector<double> to_real(const std::vector<cld>& v) {
  std::vector<double> o(v.size());
  for (size_t i = 0; i < v.size(); ++i) o[i] = static_cast<double>(v[i].real());
  return o;
}
std::vector<double> to_interleaved(const std::vector<cld>& v) {
  std::vector<double> o(2 * v.size());
  for (size_t i = 0; i < v.size(); ++i) {
    o[2 * i] = static_cast<double>(v[i].real());
    o[2 * i + 1] = static_cast<double>(v[i].imag());
  }
  return o;
}

}  // namespace

SepSolver build_sep_solver(DeviceAlloc& dev, int dim, const int* ext, const Stencil& st,
                           int time_axis_in_box, int prefer_line_axis, i64 nbatch, const std::string& what,
                           bool part_lines) {
  SepSolver s;
  s.dim = dim;
  for (int a = 0; a < 3; ++a) s.ext[a] = a < dim ? ext[a] : 1;

  // Line axis L: the time axis if present (its backward stencil is defective).  Otherwise the
  // longest axis (a dense eigenvector transform costs O(extent) per point, so the long axis
  // is the one solved by line recurrences); ties go to the slowest axis, whose lines coalesce
  // across threads.  If another axis' eigenvector scaling is too ill-conditioned it becomes L.
  auto cond_of = [&](int a) -> ld {
    const ld l = st.left[a], r = st.right[a];
    if (r == 0 || l == 0) return 1e300L;
    return std::exp(std::fabs(0.5L * std::log(std::fabs(l / r))) * static_cast<ld>(s.ext[a] - 1));
  };
  if (time_axis_in_box >= 0) {
    s.L = time_axis_in_box;
  } else if (prefer_line_axis >= 0) {
    s.L = prefer_line_axis;
  } else {
    s.L = dim - 1;
    for (int a = dim - 1; a >= 0; --a)
      if (s.ext[a] > s.ext[s.L]) s.L = a;
    int bad = -1, nbad = 0;
    for (int a = 0; a < dim; ++a)
      if (a != s.L && cond_of(a) > 1e4L) {
        bad = a;
        ++nbad;
      }
    if (nbad == 1 && cond_of(s.L) <= 1e4L) s.L = bad;
  }
  std::vector<AxisEigen> eig(3);
  for (int a = 0; a < dim; ++a) {
    if (a == s.L) continue;
    if (a == time_axis_in_box)
      throw AsdsmError(kUnsupported, what + ": the time axis cannot be diagonalized");
    s.dax[s.nd++] = a;
    eig[static_cast<size_t>(a)] = axis_eigen(s.ext[a], st.left[a], st.dpart[a], st.right[a]);
    if (eig[static_cast<size_t>(a)].cplx) s.complex_modes = true;
    if (eig[static_cast<size_t>(a)].cond > 1e4L)
      throw AsdsmError(kUnsupported, what + ": eigenvector scaling on axis " + std::to_string(a) +
                                         " too ill-conditioned for the separable solver");
  }
  if (s.complex_modes && s.nd > 1)
    throw AsdsmError(kUnsupported, what + ": complex modes on a box with two diagonalized axes");

  for (int i = 0; i < s.nd; ++i) {
    const int a = s.dax[i];
    const AxisEigen& e = eig[static_cast<size_t>(a)];
    if (s.complex_modes) {
      s.W[a] = upload(dev, to_interleaved(e.W));
      s.V[a] = upload(dev, to_interleaved(e.V));
    } else {
      s.W[a] = upload(dev, to_real(e.W));
      s.V[a] = upload(dev, to_real(e.V));
      const int m = s.ext[a];
      std::vector<double> wt(static_cast<size_t>(m) * m);
      for (int k = 0; k < m; ++k)
        for (int j = 0; j < m; ++j) wt[static_cast<size_t>(j) * m + k] = static_cast<double>(e.W[static_cast<size_t>(k) * m + j].real());
      s.Wt[a] = upload(dev, wt);
      s.half[a] = upload(dev, half_sine_tables(m, e));
    }
  }

  // Combos over the non-line axes, x fastest.
  int cext[2] = {1, 1}, cax[2] = {-1, -1}, nco = 0;
  for (int a = 0; a < dim; ++a)
    if (a != s.L) {
      cax[nco] = a;
      cext[nco] = s.ext[a];
      ++nco;
    }
  s.ncombo = cext[0] * cext[1];
  const int m = s.ext[s.L];
  const ld l = st.left[s.L], r = st.right[s.L], dL = st.dpart[s.L];
  s.line_left = st.left[s.L];
  s.line_right = st.right[s.L];
  std::vector<cld> sigma(static_cast<size_t>(s.ncombo));
  for (int c1 = 0; c1 < cext[1]; ++c1)
    for (int c0 = 0; c0 < cext[0]; ++c0) {
      cld sg = 0;
      if (cax[0] >= 0) sg += eig[static_cast<size_t>(cax[0])].lam[static_cast<size_t>(c0)];
      if (cax[1] >= 0) sg += eig[static_cast<size_t>(cax[1])].lam[static_cast<size_t>(c1)];
      sigma[static_cast<size_t>(c0 + cext[0] * c1)] = sg;
    }

  // PCR (one CTA per line) for lines along the contiguous axis or when there are few lines
  // (a per-thread Thomas walk over a few long lines is latency bound); Thomas otherwise.
  s.use_pcr = (s.L == 0) || (static_cast<i64>(s.ncombo) * nbatch < 8192 && m <= 6144);
  if (!s.use_pcr) {
    std::vector<cld> ipiv(static_cast<size_t>(m) * s.ncombo), cp(static_cast<size_t>(m) * s.ncombo);
    for (int c = 0; c < s.ncombo; ++c) {
      const cld b = cld(dL, 0) + sigma[static_cast<size_t>(c)];
      cld prev_cp = 0;
      for (int p = 0; p < m; ++p) {
        const cld w = (p == 0) ? b : b - cld(l, 0) * prev_cp;
        if (std::abs(w) == 0) throw AsdsmError(kSingularMatrix, what + ": zero pivot in a line solve");
        const cld iv = cld(1, 0) / w;
        ipiv[static_cast<size_t>(p) * s.ncombo + c] = iv;
        prev_cp = cld(r, 0) * iv;
        cp[static_cast<size_t>(p) * s.ncombo + c] = prev_cp;
      }
    }
    if (s.complex_modes) {
      s.th_ipiv = upload(dev, to_interleaved(ipiv));
      s.th_cp = upload(dev, to_interleaved(cp));
    } else {
      s.th_ipiv = upload(dev, to_real(ipiv));
      s.th_cp = upload(dev, to_real(cp));
    }
    if (part_lines && !s.complex_modes && m <= kPartMaxLine && m >= 2) build_partition_tables(s, m, l, r, dL, sigma, dev);
  } else {
    int levels = 0;
    while ((1 << levels) < m) ++levels;
    s.pcr_levels = levels;
    std::vector<cld> k1(static_cast<size_t>(s.ncombo) * levels * m), k2(k1.size()), invb(static_cast<size_t>(s.ncombo) * m);
    for (int c = 0; c < s.ncombo; ++c) {
      std::vector<cld> A(static_cast<size_t>(m), cld(l, 0)), B(static_cast<size_t>(m), cld(dL, 0) + sigma[static_cast<size_t>(c)]),
          C(static_cast<size_t>(m), cld(r, 0));
      A[0] = 0;
      C[static_cast<size_t>(m - 1)] = 0;
      for (int lev = 0, stp = 1; lev < levels; ++lev, stp <<= 1) {
        std::vector<cld> A2(A.size()), B2(B.size()), C2(C.size());
        for (int i = 0; i < m; ++i) {
          cld f1 = 0, f2 = 0;
          const bool lo = i - stp >= 0, hi = i + stp < m;
          if (lo) f1 = A[static_cast<size_t>(i)] / B[static_cast<size_t>(i - stp)];
          if (hi) f2 = C[static_cast<size_t>(i)] / B[static_cast<size_t>(i + stp)];
          A2[static_cast<size_t>(i)] = lo ? -A[static_cast<size_t>(i - stp)] * f1 : cld(0);
          C2[static_cast<size_t>(i)] = hi ? -C[static_cast<size_t>(i + stp)] * f2 : cld(0);
          B2[static_cast<size_t>(i)] = B[static_cast<size_t>(i)] - (lo ? C[static_cast<size_t>(i - stp)] * f1 : cld(0)) -
                                      (hi ? A[static_cast<size_t>(i + stp)] * f2 : cld(0));
          k1[(static_cast<size_t>(c) * levels + lev) * m + i] = f1;
          k2[(static_cast<size_t>(c) * levels + lev) * m + i] = f2;
        }
        A.swap(A2);
        B.swap(B2);
        C.swap(C2);
      }
      for (int i = 0; i < m; ++i) {
        if (std::abs(B[static_cast<size_t>(i)]) == 0) throw AsdsmError(kSingularMatrix, what + ": zero pivot in PCR");
        invb[static_cast<size_t>(c) * m + i] = cld(1, 0) / B[static_cast<size_t>(i)];
      }
    }
    if (!s.complex_modes && m <= kPartMaxLine && m >= 2) build_partition_tables(s, m, l, r, dL, sigma, dev);
    if (s.complex_modes) {
      s.pcr_k1 = upload(dev, to_interleaved(k1));
      s.pcr_k2 = upload(dev, to_interleaved(k2));
      s.pcr_invb = upload(dev, to_interleaved(invb));
    } else {
      s.pcr_k1 = upload(dev, to_real(k1));
      s.pcr_k2 = upload(dev, to_real(k2));
      s.pcr_invb = upload(dev, to_real(invb));
    }
  }
  return s;
}

}  // namespace asdsm_b200
