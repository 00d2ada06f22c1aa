// Host-side right-hand-side assembly: the reference's rhs_core (proj/src/fdm.cpp:128-171)
// for any tensor kind, same sampling coordinates and lifting order.  Runs once per problem
// (setup), parallel over rows with std::thread; the solve itself never comes back here.
#include "assemble.hpp"

#include <algorithm>
#include <thread>
#include <vector>

namespace asdsm_b200 {

void assemble_rhs(const Mesh& m, unsigned mask, const asdsm_cat::Problem& p, double* out) {
  const int dim = m.dim;
  int count[3] = {1, 1, 1}, stride[3] = {1, 1, 1};
  for (int a = 0; a < dim; ++a) {
    const bool coarse = (mask >> a) & 1u;
    count[a] = coarse ? m.nc[a] : m.nf[a];
    stride[a] = coarse ? m.n[a] : 1;
  }
  const i64 rows = static_cast<i64>(count[1]) * (dim == 3 ? count[2] : 1);
  auto work = [&](i64 r0, i64 r1) {
    for (i64 row = r0; row < r1; ++row) {
      int idx[3] = {1, static_cast<int>(row % count[1]) + 1, dim == 3 ? static_cast<int>(row / count[1]) + 1 : 1};
      for (int i = 1; i <= count[0]; ++i) {
        idx[0] = i;
        asdsm_cat::Coord x{0.0, 0.0, 0.0};
        for (int a = 0; a < dim; ++a)
          x[static_cast<size_t>(a)] = static_cast<double>(static_cast<i64>(idx[a]) * stride[a]) * m.h[a];
        double v = p.source(x);
        for (int a = 0; a < dim; ++a) {
          const bool coarse = (mask >> a) & 1u;
          const double step = coarse ? m.H[a] : m.h[a];
          double left, right;
          bool has_right = true;
          if (a == m.time_axis) {
            const double tc = 1.0 / step;
            left = -tc;
            right = 0.0;
            has_right = false;
          } else {
            const double al = p.alpha[static_cast<size_t>(a)](x);
            const double c = al / (step * step);
            const double d = p.beta[static_cast<size_t>(a)](x) / (2.0 * step);
            left = -c - d;
            right = -c + d;
          }
          if (idx[a] == 1) {
            asdsm_cat::Coord xb = x;
            xb[static_cast<size_t>(a)] = static_cast<double>(0) * m.h[a];
            v -= left * p.boundary(xb);
          }
          if (idx[a] == count[a] && has_right) {
            asdsm_cat::Coord xb = x;
            xb[static_cast<size_t>(a)] = static_cast<double>(static_cast<i64>(count[a] + 1) * stride[a]) * m.h[a];
            v -= right * p.boundary(xb);
          }
        }
        out[(idx[0] - 1) + static_cast<i64>(count[0]) * row] = v;
      }
    }
  };
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const i64 nt = std::min<i64>(hw, rows);
  if (nt <= 1 || static_cast<i64>(count[0]) * rows < 100000) {
    work(0, rows);
    return;
  }
  std::vector<std::thread> th;
  for (i64 t = 0; t < nt; ++t) th.emplace_back(work, rows * t / nt, rows * (t + 1) / nt);
  for (auto& t : th) t.join();
}

void sample_exact(const Mesh& m, const asdsm_cat::Problem& p, double* out) {
  const int dim = m.dim;
  const i64 rows = static_cast<i64>(m.nf[1]) * (dim == 3 ? m.nf[2] : 1);
  auto work = [&](i64 r0, i64 r1) {
    for (i64 row = r0; row < r1; ++row) {
      const int j = static_cast<int>(row % m.nf[1]) + 1;
      const int k = dim == 3 ? static_cast<int>(row / m.nf[1]) + 1 : 0;
      for (int i = 1; i <= m.nf[0]; ++i) {
        asdsm_cat::Coord x{static_cast<double>(i) * m.h[0], static_cast<double>(j) * m.h[1],
                           dim == 3 ? static_cast<double>(k) * m.h[2] : 0.0};
        out[(i - 1) + static_cast<i64>(m.nf[0]) * row] = p.exact(x);
      }
    }
  };
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const i64 nt = std::min<i64>(hw, rows);
  std::vector<std::thread> th;
  for (i64 t = 0; t < nt; ++t) th.emplace_back(work, rows * t / nt, rows * (t + 1) / nt);
  for (auto& t : th) t.join();
}

bool uniform_coefficients(const Mesh& m, const asdsm_cat::Problem& p, double* alpha, double* beta) {
  const int dim = m.dim;
  for (int a = 0; a < 3; ++a) alpha[a] = beta[a] = 0.0;
  asdsm_cat::Coord x0{0.0, 0.0, 0.0};
  for (int a = 0; a < dim; ++a) x0[static_cast<size_t>(a)] = m.h[a];
  for (int a = 0; a < dim; ++a) {
    if (a == m.time_axis) continue;
    alpha[a] = p.alpha[static_cast<size_t>(a)](x0);
    beta[a] = p.beta[static_cast<size_t>(a)](x0);
  }
  const i64 rows = static_cast<i64>(m.nf[1]) * (dim == 3 ? m.nf[2] : 1);
  std::vector<char> ok(static_cast<size_t>(rows), 1), pos(static_cast<size_t>(rows), 1);
  auto work = [&](i64 r0, i64 r1) {
    for (i64 row = r0; row < r1; ++row) {
      const int j = static_cast<int>(row % m.nf[1]) + 1;
      const int k = dim == 3 ? static_cast<int>(row / m.nf[1]) + 1 : 0;
      for (int i = 1; i <= m.nf[0]; ++i) {
        asdsm_cat::Coord x{static_cast<double>(i) * m.h[0], static_cast<double>(j) * m.h[1],
                           dim == 3 ? static_cast<double>(k) * m.h[2] : 0.0};
        for (int a = 0; a < dim; ++a) {
          if (a == m.time_axis) continue;
          const double al = p.alpha[static_cast<size_t>(a)](x);
          if (!(al > 0.0)) pos[static_cast<size_t>(row)] = 0;
          if (al != alpha[a] || p.beta[static_cast<size_t>(a)](x) != beta[a]) ok[static_cast<size_t>(row)] = 0;
        }
      }
    }
  };
  const unsigned hw = std::max(1u, std::min(32u, std::thread::hardware_concurrency()));
  const i64 nt = std::min<i64>(hw, rows);
  if (nt <= 1 || static_cast<i64>(m.nf[0]) * rows < 100000) {
    work(0, rows);
  } else {
    std::vector<std::thread> th;
    for (i64 t = 0; t < nt; ++t) th.emplace_back(work, rows * t / nt, rows * (t + 1) / nt);
    for (auto& t : th) t.join();
  }
  for (char c : pos)
    if (!c) throw AsdsmError(kError, "diffusion coefficient not positive");
  for (char c : ok)
    if (!c) return false;
  return true;
}

}  // namespace asdsm_b200
