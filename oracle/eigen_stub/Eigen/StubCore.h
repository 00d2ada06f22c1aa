// Eigen stand-in core for oracle/_ref (test infrastructure only, never shipped).
//
// Reference dependency replaced: Eigen 3.3+ SparseLU (supernodal sparse LU with COLAMD
// fill-reducing column ordering and partial pivoting, diagonal pivot threshold 1.0).
// Published algorithm restated here: sparse LU with partial (row) pivoting after a
// fill-reducing symmetric reordering.  This stand-in uses reverse Cuthill-McKee for the
// ordering (instead of COLAMD) and a LAPACK-dgbtf2-style band LU with partial pivoting.
// The factorization is the same mathematical object (P A Q = L U up to the ordering), so
// solves agree with Eigen's to rounding; the rounding itself differs.
#pragma once
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <vector>

namespace Eigen {

enum ComputationInfo { Success = 0, NumericalIssue = 1, InvalidInput = 3 };
using Index = std::ptrdiff_t;

template <typename Scalar>
struct Triplet {
  Triplet(int r, int c, Scalar v) : r_(r), c_(c), v_(v) {}
  int row() const { return r_; }
  int col() const { return c_; }
  Scalar value() const { return v_; }
  int r_, c_;
  Scalar v_;
};

class VectorXd {
 public:
  VectorXd() = default;
  explicit VectorXd(Index n) : d_(static_cast<std::size_t>(n), 0.0) {}
  double& operator[](Index i) { return d_[static_cast<std::size_t>(i)]; }
  double operator[](Index i) const { return d_[static_cast<std::size_t>(i)]; }
  double* data() { return d_.data(); }
  const double* data() const { return d_.data(); }
  Index size() const { return static_cast<Index>(d_.size()); }

 private:
  std::vector<double> d_;
};

template <typename Scalar>
class SparseMatrix {
 public:
  SparseMatrix(Index rows, Index cols) : rows_(rows), cols_(cols) {}
  template <typename It>
  void setFromTriplets(It begin, It end) {
    for (It it = begin; it != end; ++it) ent_.push_back({it->row(), it->col(), it->value()});
    std::sort(ent_.begin(), ent_.end(), [](const E& a, const E& b) {
      return a.r != b.r ? a.r < b.r : a.c < b.c;
    });
    // Duplicates are summed, as Eigen does.
    std::vector<E> merged;
    for (const E& e : ent_) {
      if (!merged.empty() && merged.back().r == e.r && merged.back().c == e.c)
        merged.back().v += e.v;
      else
        merged.push_back(e);
    }
    ent_ = std::move(merged);
  }
  void makeCompressed() {}
  Index rows() const { return rows_; }
  Index cols() const { return cols_; }

  struct E {
    int r, c;
    Scalar v;
  };
  const std::vector<E>& entries() const { return ent_; }

 private:
  Index rows_, cols_;
  std::vector<E> ent_;
};

template <typename I>
struct COLAMDOrdering {};

template <typename MatrixType, typename Ordering>
class SparseLU {
 public:
  void analyzePattern(const MatrixType& m) {
    n_ = m.rows();
    info_ = Success;
    if (m.rows() != m.cols()) {
      info_ = InvalidInput;
      msg_ = "matrix is not square";
      return;
    }
    // Symmetrized adjacency for the reverse Cuthill-McKee ordering.
    std::vector<std::vector<int>> adj(static_cast<std::size_t>(n_));
    for (const auto& e : m.entries())
      if (e.r != e.c) {
        adj[static_cast<std::size_t>(e.r)].push_back(e.c);
        adj[static_cast<std::size_t>(e.c)].push_back(e.r);
      }
    for (auto& a : adj) {
      std::sort(a.begin(), a.end());
      a.erase(std::unique(a.begin(), a.end()), a.end());
    }
    perm_.clear();
    std::vector<char> seen(static_cast<std::size_t>(n_), 0);
    for (Index start0 = 0; start0 < n_; ++start0) {
      if (seen[static_cast<std::size_t>(start0)]) continue;
      // Pseudo-peripheral start: the minimum-degree node of this component found by BFS.
      int start = static_cast<int>(start0);
      {
        std::vector<int> comp{start};
        std::vector<char> mark(static_cast<std::size_t>(n_), 0);
        mark[static_cast<std::size_t>(start)] = 1;
        for (std::size_t q = 0; q < comp.size(); ++q)
          for (int nb : adj[static_cast<std::size_t>(comp[q])])
            if (!mark[static_cast<std::size_t>(nb)]) {
              mark[static_cast<std::size_t>(nb)] = 1;
              comp.push_back(nb);
            }
        for (int v : comp)
          if (adj[static_cast<std::size_t>(v)].size() < adj[static_cast<std::size_t>(start)].size() ||
              (adj[static_cast<std::size_t>(v)].size() == adj[static_cast<std::size_t>(start)].size() && v < start))
            start = v;
      }
      std::vector<int> level{start};
      seen[static_cast<std::size_t>(start)] = 1;
      for (std::size_t q = 0; q < level.size(); ++q) {
        std::vector<int> nbs;
        for (int nb : adj[static_cast<std::size_t>(level[q])])
          if (!seen[static_cast<std::size_t>(nb)]) {
            seen[static_cast<std::size_t>(nb)] = 1;
            nbs.push_back(nb);
          }
        std::sort(nbs.begin(), nbs.end(), [&](int a, int b) {
          const auto da = adj[static_cast<std::size_t>(a)].size(), db = adj[static_cast<std::size_t>(b)].size();
          return da != db ? da < db : a < b;
        });
        level.insert(level.end(), nbs.begin(), nbs.end());
      }
      if (const char* o = std::getenv("ASDSM_STUB_ORDER"); o && std::string(o) == "cm")
        perm_.insert(perm_.end(), level.begin(), level.end());  // Cuthill-McKee, not reversed
      else
        perm_.insert(perm_.end(), level.rbegin(), level.rend());
    }
    if (std::getenv("ASDSM_STUB_NATURAL_ORDER")) {
      perm_.resize(static_cast<std::size_t>(n_));
      for (Index k = 0; k < n_; ++k) perm_[static_cast<std::size_t>(k)] = static_cast<int>(k);
    }
    inv_.assign(static_cast<std::size_t>(n_), 0);
    for (Index k = 0; k < n_; ++k) inv_[static_cast<std::size_t>(perm_[static_cast<std::size_t>(k)])] = static_cast<int>(k);
    bw_ = 0;
    for (const auto& e : m.entries())
      bw_ = std::max<Index>(bw_, std::abs(inv_[static_cast<std::size_t>(e.r)] - inv_[static_cast<std::size_t>(e.c)]));
  }

  void factorize(const MatrixType& m) {
    if (info_ != Success) return;
    kl_ = bw_;
    ku_ = bw_;
    kv_ = kl_ + ku_;
    ld_ = 2 * kl_ + ku_ + 1;
    ab_.assign(static_cast<std::size_t>(ld_ * n_), 0.0);
    for (const auto& e : m.entries()) {
      const Index r = inv_[static_cast<std::size_t>(e.r)], c = inv_[static_cast<std::size_t>(e.c)];
      at(r, c) = e.v;
    }
    ipiv_.assign(static_cast<std::size_t>(n_), 0);
    Index ju = 0;
    for (Index j = 0; j < n_; ++j) {
      const Index km = std::min(kl_, n_ - 1 - j);
      Index jp = 0;
      double best = std::abs(at(j, j));
      for (Index i = 1; i <= km; ++i)
        if (std::abs(at(j + i, j)) > best) {
          best = std::abs(at(j + i, j));
          jp = i;
        }
      ipiv_[static_cast<std::size_t>(j)] = j + jp;
      if (!(best > 0.0)) {
        info_ = NumericalIssue;
        msg_ = "zero pivot in column " + std::to_string(j);
        return;
      }
      ju = std::max(ju, std::min(j + ku_ + jp, n_ - 1));
      if (jp != 0)
        for (Index c = j; c <= ju; ++c) std::swap(at(j, c), at(j + jp, c));
      const double piv = at(j, j);
      for (Index i = 1; i <= km; ++i) at(j + i, j) /= piv;
      for (Index c = j + 1; c <= ju; ++c) {
        const double t = at(j, c);
        if (t != 0.0) {
          double* col = &at(j + 1, c);
          const double* l = &at(j + 1, j);
          for (Index i = 0; i < km; ++i) col[i] -= l[i] * t;
        }
      }
    }
  }

  ComputationInfo info() const { return info_; }
  std::string lastErrorMessage() const { return msg_; }

  VectorXd solve(const VectorXd& rhs) const {
    VectorXd x(n_);
    std::vector<double> b(static_cast<std::size_t>(n_));
    for (Index k = 0; k < n_; ++k) b[static_cast<std::size_t>(k)] = rhs[perm_[static_cast<std::size_t>(k)]];
    for (Index j = 0; j < n_; ++j) {
      const Index p = ipiv_[static_cast<std::size_t>(j)];
      if (p != j) std::swap(b[static_cast<std::size_t>(j)], b[static_cast<std::size_t>(p)]);
      const double bj = b[static_cast<std::size_t>(j)];
      const Index km = std::min(kl_, n_ - 1 - j);
      if (bj != 0.0)
        for (Index i = 1; i <= km; ++i) b[static_cast<std::size_t>(j + i)] -= at(j + i, j) * bj;
    }
    for (Index j = n_ - 1; j >= 0; --j) {
      b[static_cast<std::size_t>(j)] /= at(j, j);
      const double bj = b[static_cast<std::size_t>(j)];
      if (bj != 0.0)
        for (Index i = std::max<Index>(0, j - kv_); i < j; ++i) b[static_cast<std::size_t>(i)] -= at(i, j) * bj;
    }
    for (Index k = 0; k < n_; ++k) x[perm_[static_cast<std::size_t>(k)]] = b[static_cast<std::size_t>(k)];
    return x;
  }

 private:
  double& at(Index r, Index c) { return ab_[static_cast<std::size_t>(kv_ + r - c + c * ld_)]; }
  double at(Index r, Index c) const { return ab_[static_cast<std::size_t>(kv_ + r - c + c * ld_)]; }

  Index n_ = 0, bw_ = 0, kl_ = 0, ku_ = 0, kv_ = 0, ld_ = 1;
  std::vector<int> perm_, inv_;
  std::vector<double> ab_;
  std::vector<Index> ipiv_;
  ComputationInfo info_ = Success;
  std::string msg_;
};

}  // namespace Eigen
