// Host side of the variable-coefficient path: coefficient sampling (fdm.cpp:63-126) and
// block-Thomas factorizations (long double Gauss-Jordan with partial pivoting per block).
#include "varcoef.hpp"

#include <algorithm>
#include <cmath>
#include <stdexcept>
#include <thread>

namespace asdsm_b200 {

using ld = long double;

std::vector<double> sample_kind_coefficients(const Mesh& m, unsigned mask, const asdsm_cat::Problem& p) {
  const int D = m.dim;
  const int ns = 2 * D + 1;
  int ext[3] = {1, 1, 1}, stride[3] = {1, 1, 1};
  for (int a = 0; a < D; ++a) {
    const bool c = (mask >> a) & 1u;
    ext[a] = c ? m.nc[a] : m.nf[a];
    stride[a] = c ? m.n[a] : 1;
  }
  const i64 n = static_cast<i64>(ext[0]) * ext[1] * ext[2];
  std::vector<double> coef(static_cast<size_t>(ns) * n, 0.0);
  auto work = [&](i64 p0, i64 p1) {
    for (i64 lin = p0; lin < p1; ++lin) {
      int idx[3] = {static_cast<int>(lin % ext[0]), static_cast<int>((lin / ext[0]) % ext[1]),
                    static_cast<int>(lin / (static_cast<i64>(ext[0]) * ext[1]))};
      asdsm_cat::Coord x{0.0, 0.0, 0.0};
      for (int a = 0; a < D; ++a)
        x[static_cast<size_t>(a)] = static_cast<double>(static_cast<i64>(idx[a] + 1) * stride[a]) * m.h[a];
      double diag = 0.0, left[3] = {0, 0, 0}, right[3] = {0, 0, 0};
      for (int a = 0; a < D; ++a) {
        const bool c = (mask >> a) & 1u;
        const double step = c ? m.H[a] : m.h[a];
        if (a == m.time_axis) {
          const double tc = 1.0 / step;
          diag += tc;
          left[a] = -tc;
          right[a] = 0.0;
          continue;
        }
        const double al = p.alpha[static_cast<size_t>(a)](x);
        if (!(al > 0.0)) throw AsdsmError(kError, "diffusion coefficient not positive on axis " + std::to_string(a));
        const double cc = al / (step * step);
        const double d = p.beta[static_cast<size_t>(a)](x) / (2.0 * step);
        diag += 2.0 * cc;
        left[a] = -cc - d;
        right[a] = -cc + d;
      }
      int s = 0;
      for (int a = D - 1; a >= 0; --a) coef[static_cast<size_t>(s++) * n + lin] = idx[a] > 0 ? left[a] : 0.0;
      coef[static_cast<size_t>(s++) * n + lin] = diag;
      for (int a = 0; a < D; ++a)
        coef[static_cast<size_t>(s++) * n + lin] = (idx[a] < ext[a] - 1 && a != m.time_axis) ? right[a] : 0.0;
    }
  };
  const i64 nt = std::min<i64>(std::max(1u, std::thread::hardware_concurrency()), 32);
  if (n < 65536 || nt <= 1) {
    work(0, n);
  } else {
    std::vector<std::thread> th;
    for (i64 t = 0; t < nt; ++t) th.emplace_back(work, n * t / nt, n * (t + 1) / nt);
    for (auto& t : th) t.join();
  }
  return coef;
}

namespace {

// In-place inverse of a B x B row-major matrix (long double, partial pivoting).
void invert(std::vector<ld>& A, int B, const std::string& what) {
  std::vector<ld> I(static_cast<size_t>(B) * B, 0.0L);
  for (int i = 0; i < B; ++i) I[static_cast<size_t>(i) * B + i] = 1.0L;
  for (int c = 0; c < B; ++c) {
    int piv = c;
    ld best = std::fabs(A[static_cast<size_t>(c) * B + c]);
    for (int r = c + 1; r < B; ++r)
      if (std::fabs(A[static_cast<size_t>(r) * B + c]) > best) {
        best = std::fabs(A[static_cast<size_t>(r) * B + c]);
        piv = r;
      }
    if (!(best > 0.0L)) throw AsdsmError(kSingularMatrix, what + ": singular block");
    if (piv != c)
      for (int k = 0; k < B; ++k) {
        std::swap(A[static_cast<size_t>(c) * B + k], A[static_cast<size_t>(piv) * B + k]);
        std::swap(I[static_cast<size_t>(c) * B + k], I[static_cast<size_t>(piv) * B + k]);
      }
    const ld inv = 1.0L / A[static_cast<size_t>(c) * B + c];
    for (int k = 0; k < B; ++k) {
      A[static_cast<size_t>(c) * B + k] *= inv;
      I[static_cast<size_t>(c) * B + k] *= inv;
    }
    for (int r = 0; r < B; ++r) {
      if (r == c) continue;
      const ld f = A[static_cast<size_t>(r) * B + c];
      if (f == 0.0L) continue;
      for (int k = 0; k < B; ++k) {
        A[static_cast<size_t>(r) * B + k] -= f * A[static_cast<size_t>(c) * B + k];
        I[static_cast<size_t>(r) * B + k] -= f * I[static_cast<size_t>(c) * B + k];
      }
    }
  }
  A.swap(I);
}

}  // namespace

template <typename F>
void factor_block_thomas(BlockThomas& bt, int nboxes, F coef) {
  const int D = bt.dim;
  const int B = bt.B, nb = bt.nb, L = bt.L;
  int oax[2] = {-1, -1}, no = 0;
  for (int a = 0; a < D; ++a)
    if (a != L) oax[no++] = a;
  i64 lstride[3] = {1, 1, 1};
  lstride[1] = bt.ext[0];
  lstride[2] = static_cast<i64>(bt.ext[0]) * bt.ext[1];
  bt.dinv.assign(static_cast<size_t>(nboxes) * nb * B * B, 0.0);
  bt.lo.assign(static_cast<size_t>(nboxes) * nb * B, 0.0);
  bt.up.assign(static_cast<size_t>(nboxes) * nb * B, 0.0);
  auto point = [&](int j, int q) -> i64 {  // box-local linear index of in-plane q in block j
    int idx[3] = {0, 0, 0};
    idx[L] = j;
    idx[oax[0]] = q % bt.ext[oax[0]];
    if (no > 1) idx[oax[1]] = q / bt.ext[oax[0]];
    return idx[0] + lstride[1] * idx[1] + lstride[2] * idx[2];
  };
  auto work = [&](int b0, int b1) {
    std::vector<ld> S(static_cast<size_t>(B) * B), prev(static_cast<size_t>(B) * B);
    for (int box = b0; box < b1; ++box) {
      for (int j = 0; j < nb; ++j) {
        std::fill(S.begin(), S.end(), 0.0L);
        for (int q = 0; q < B; ++q) {
          const i64 p = point(j, q);
          int idx[3] = {static_cast<int>(p % bt.ext[0]), static_cast<int>((p / bt.ext[0]) % bt.ext[1]),
                        static_cast<int>(p / lstride[2])};
          // slot order: left[D-1..0], diag, right[0..D-1]
          S[static_cast<size_t>(q) * B + q] = coef(box, p, D);
          for (int oi = 0; oi < no; ++oi) {
            const int a = oax[oi];
            const int qs = oi == 0 ? 1 : bt.ext[oax[0]];
            if (idx[a] > 0) S[static_cast<size_t>(q) * B + (q - qs)] = coef(box, p, D - 1 - a);
            if (idx[a] < bt.ext[a] - 1) S[static_cast<size_t>(q) * B + (q + qs)] = coef(box, p, D + 1 + a);
          }
          const double lj = j > 0 ? coef(box, p, D - 1 - L) : 0.0;
          const double rj = j < nb - 1 ? coef(box, p, D + 1 + L) : 0.0;
          bt.lo[(static_cast<size_t>(box) * nb + j) * B + q] = lj;
          bt.up[(static_cast<size_t>(box) * nb + j) * B + q] = rj;
        }
        if (j > 0) {  // S_j = A_jj - diag(l_j) S_{j-1}^{-1} diag(r_{j-1})
          for (int p = 0; p < B; ++p) {
            const ld lj = bt.lo[(static_cast<size_t>(box) * nb + j) * B + p];
            if (lj == 0.0L) continue;
            for (int q = 0; q < B; ++q) {
              const ld rq = bt.up[(static_cast<size_t>(box) * nb + j - 1) * B + q];
              S[static_cast<size_t>(p) * B + q] -= lj * prev[static_cast<size_t>(p) * B + q] * rq;
            }
          }
        }
        invert(S, B, "block-Thomas factor");
        prev = S;
        double* dst = bt.dinv.data() + (static_cast<size_t>(box) * nb + j) * B * B;
        for (int i = 0; i < B; ++i)
          for (int k = 0; k < B; ++k) dst[static_cast<size_t>(k) * B + i] = static_cast<double>(S[static_cast<size_t>(i) * B + k]);
      }
    }
  };
  const int nt = static_cast<int>(std::min<unsigned>(std::max(1u, std::thread::hardware_concurrency()), 32u));
  if (nboxes < 4 || nt <= 1) {
    work(0, nboxes);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t) th.emplace_back(work, nboxes * t / nt, nboxes * (t + 1) / nt);
    for (auto& t : th) t.join();
  }
}

static void choose_axis(BlockThomas& bt, int time_axis) {
  // longest axis (ties: slowest) carries the blocks; the time axis has no right coupling but
  // block Thomas handles it like any other axis
  (void)time_axis;
  bt.L = bt.dim - 1;
  for (int a = bt.dim - 1; a >= 0; --a)
    if (bt.ext[a] > bt.ext[bt.L]) bt.L = a;
  bt.nb = bt.ext[bt.L];
  bt.B = 1;
  for (int a = 0; a < bt.dim; ++a)
    if (a != bt.L) bt.B *= bt.ext[a];
  if (bt.B > 1024) throw AsdsmError(kUnsupported, "variable-coefficient block size above 1024");
}

BlockThomas factor_kind_box(const Mesh& m, unsigned mask, const std::vector<double>& coef, int time_axis) {
  BlockThomas bt;
  bt.dim = m.dim;
  for (int a = 0; a < 3; ++a) bt.ext[a] = a < m.dim ? m.axis_points(mask, a) : 1;
  choose_axis(bt, time_axis);
  const i64 n = static_cast<i64>(bt.ext[0]) * bt.ext[1] * bt.ext[2];
  factor_block_thomas(bt, 1, [&](int, i64 p, int slot) { return coef[static_cast<size_t>(slot) * n + p]; });
  return bt;
}

BlockThomas factor_hole_boxes(const Mesh& m, const std::vector<double>& fine_coef) {
  BlockThomas bt;
  bt.dim = m.dim;
  int nbox[3] = {1, 1, 1};
  for (int a = 0; a < 3; ++a) {
    bt.ext[a] = a < m.dim ? m.n[a] - 1 : 1;
    nbox[a] = a < m.dim ? m.nc[a] + 1 : 1;
  }
  choose_axis(bt, m.time_axis);
  const i64 N = m.point_count(0u);
  const int nboxes = nbox[0] * nbox[1] * nbox[2];
  factor_block_thomas(bt, nboxes, [&](int box, i64 p, int slot) {
    const int hx = box % nbox[0], hy = (box / nbox[0]) % nbox[1], hz = box / (nbox[0] * nbox[1]);
    const int i = static_cast<int>(p % bt.ext[0]), j = static_cast<int>((p / bt.ext[0]) % bt.ext[1]),
              k = static_cast<int>(p / (static_cast<i64>(bt.ext[0]) * bt.ext[1]));
    const i64 fx = static_cast<i64>(hx) * m.n[0] + i, fy = static_cast<i64>(hy) * m.n[1] + j,
              fz = m.dim == 3 ? static_cast<i64>(hz) * m.n[2] + k : 0;
    const i64 f = fx + m.nf[0] * (fy + static_cast<i64>(m.nf[1]) * fz);
    return fine_coef[static_cast<size_t>(slot) * N + f];
  });
  return bt;
}

}  // namespace asdsm_b200
