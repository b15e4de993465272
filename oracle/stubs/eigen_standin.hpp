// Minimal stand-in for the three Eigen headers the reference includes.
//
// TEST INFRASTRUCTURE (oracle/).  Eigen3 is a third-party dependency of the
// reference (find_package(Eigen3 3.3 REQUIRED), proj/core/CMakeLists.txt:1;
// version not pinned) that is absent from this image.  The reference uses it
// in exactly two places:
//   * Eigen::SparseLU<SparseMatrix<double,ColMajor,int>> in
//     proj/core/src/linalg.cpp:76-104 (the G_x factor for n_x > 64), built
//     with default template arguments: COLAMDOrdering and a diagonal pivot
//     threshold of 1.0, i.e. partial pivoting (Eigen 3.3+ documented defaults);
//   * Eigen::AMDOrdering in proj/core/src/sparse_ldlt.cpp:14-28 (augmented
//     strategy only; the reduced path reaches it only on its fallback).
// This header restates the published algorithms, not Eigen's code:
//   * column ordering: minimum degree on the pattern of A'A (the quantity
//     COLAMD approximates), ties broken by lowest index;
//   * numeric factor: left-looking Gilbert-Peierls sparse LU with partial
//     pivoting (largest magnitude in the column; diagonal preferred on ties),
//     P A Q = L U with unit-diagonal L; factorize() reports NumericalIssue iff
//     a zero pivot is met, which is when Eigen's SparseLU fails;
//   * AMD: exact minimum degree on A + A' (a valid fill-reducing order; only
//     the augmented fallback uses it).
// Results agree with Eigen's to rounding (same factorisation family); the
// ordering and therefore fill differ.  Every report built on this oracle says
// so (bench.py cpu_baseline.sample).
#pragma once

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <set>
#include <stdexcept>
#include <utility>
#include <vector>

namespace Eigen {

enum StorageOptions { ColMajor = 0, RowMajor = 1 };
enum UpLoType { Lower = 1, Upper = 2 };
constexpr int Dynamic = -1;
enum ComputationInfo { Success = 0, NumericalIssue = 1, NoConvergence = 2, InvalidInput = 3 };

template <typename Scalar, typename Index = int>
struct Triplet {
  Index r = 0, c = 0;
  Scalar v = 0;
  Triplet() = default;
  Triplet(Index row, Index col, Scalar value) : r(row), c(col), v(value) {}
  Index row() const { return r; }
  Index col() const { return c; }
  Scalar value() const { return v; }
};

template <typename MatrixType, int UpLo>
struct SelfAdjointView {
  const MatrixType& m;
};

// Compressed-column sparse matrix; duplicates are summed (as Eigen does).
template <typename Scalar, int Options = ColMajor, typename Index = int>
class SparseMatrix {
 public:
  SparseMatrix() = default;
  SparseMatrix(Index rows, Index cols) : rows_(rows), cols_(cols), colptr_(size_t(cols) + 1, 0) {}

  template <typename It>
  void setFromTriplets(It begin, It end) {
    std::vector<std::pair<std::pair<Index, Index>, Scalar>> t;
    for (It it = begin; it != end; ++it) t.push_back({{it->col(), it->row()}, it->value()});
    std::stable_sort(t.begin(), t.end(),
                     [](const auto& a, const auto& b) { return a.first < b.first; });
    colptr_.assign(size_t(cols_) + 1, 0);
    rowind_.clear();
    val_.clear();
    for (size_t k = 0; k < t.size(); ++k) {
      if (k > 0 && t[k].first == t[k - 1].first) {
        val_.back() += t[k].second;
        continue;
      }
      colptr_[size_t(t[k].first.first) + 1]++;
      rowind_.push_back(t[k].first.second);
      val_.push_back(t[k].second);
    }
    for (Index j = 0; j < cols_; ++j) colptr_[size_t(j) + 1] += colptr_[size_t(j)];
  }

  template <int UpLo>
  SelfAdjointView<SparseMatrix, UpLo> selfadjointView() const {
    return {*this};
  }

  Index rows() const { return rows_; }
  Index cols() const { return cols_; }
  const std::vector<Index>& colptr() const { return colptr_; }
  const std::vector<Index>& rowind() const { return rowind_; }
  const std::vector<Scalar>& values() const { return val_; }

 private:
  Index rows_ = 0, cols_ = 0;
  std::vector<Index> colptr_, rowind_;
  std::vector<Scalar> val_;
};

class MatrixXd;

template <typename T>
class Map;

// Dense column-major matrix (only what the reference's call sites need).
class MatrixXd {
 public:
  MatrixXd() = default;
  MatrixXd(long rows, long cols) : rows_(rows), cols_(cols), a_(size_t(rows * cols), 0.0) {}
  inline MatrixXd(const Map<MatrixXd>& m);
  long rows() const { return rows_; }
  long cols() const { return cols_; }
  double* data() { return a_.data(); }
  const double* data() const { return a_.data(); }
  MatrixXd eval() const { return *this; }

 private:
  long rows_ = 0, cols_ = 0;
  std::vector<double> a_;
};

template <>
class Map<MatrixXd> {
 public:
  Map(double* p, long rows, long cols) : p_(p), rows_(rows), cols_(cols) {}
  Map& operator=(const MatrixXd& m) {
    if (m.rows() != rows_ || m.cols() != cols_) throw std::runtime_error("Map: shape mismatch");
    std::copy(m.data(), m.data() + rows_ * cols_, p_);
    return *this;
  }
  long rows() const { return rows_; }
  long cols() const { return cols_; }
  const double* data() const { return p_; }

 private:
  double* p_;
  long rows_, cols_;
};

inline MatrixXd::MatrixXd(const Map<MatrixXd>& m)
    : rows_(m.rows()), cols_(m.cols()), a_(m.data(), m.data() + m.rows() * m.cols()) {}

template <int Size, int MaxSize, typename Index>
class PermutationMatrix {
 public:
  struct Indices {
    std::vector<Index> v;
    Index* data() { return v.data(); }
    const Index* data() const { return v.data(); }
    Index size() const { return Index(v.size()); }
  };
  Indices& indices() { return ind_; }
  const Indices& indices() const { return ind_; }

 private:
  Indices ind_;
};

namespace standin {

// Exact minimum degree on a symmetric adjacency structure (no self loops).
// Returns the elimination order; ties go to the lowest index.
inline std::vector<int> minimum_degree(std::vector<std::vector<int>> adj) {
  const int n = int(adj.size());
  std::vector<char> gone(size_t(n), 0);
  std::set<std::pair<int, int>> q;
  for (int i = 0; i < n; ++i) q.insert({int(adj[size_t(i)].size()), i});
  std::vector<int> order;
  order.reserve(static_cast<size_t>(n));
  std::vector<int> merged;
  while (!q.empty()) {
    const int v = q.begin()->second;
    q.erase(q.begin());
    gone[size_t(v)] = 1;
    order.push_back(v);
    std::vector<int> nb;
    for (int u : adj[size_t(v)])
      if (!gone[size_t(u)]) nb.push_back(u);
    for (int u : nb) {
      auto& au = adj[size_t(u)];
      q.erase({int(au.size()), u});
      merged.clear();
      std::set_union(au.begin(), au.end(), nb.begin(), nb.end(), std::back_inserter(merged));
      au.clear();
      for (int w : merged)
        if (w != u && !gone[size_t(w)]) au.push_back(w);
      q.insert({int(au.size()), u});
    }
    adj[size_t(v)].clear();
  }
  return order;
}

}  // namespace standin

template <typename Index>
class AMDOrdering {
 public:
  template <typename MatrixType, int UpLo>
  void operator()(const SelfAdjointView<MatrixType, UpLo>& sa,
                  PermutationMatrix<Dynamic, Dynamic, Index>& perm) const {
    const auto& m = sa.m;
    const int n = int(m.cols());
    std::vector<std::vector<int>> adj(static_cast<size_t>(n));
    for (int j = 0; j < n; ++j)
      for (Index k = m.colptr()[size_t(j)]; k < m.colptr()[size_t(j) + 1]; ++k) {
        const int i = int(m.rowind()[size_t(k)]);
        if (i == j) continue;
        adj[size_t(i)].push_back(j);
        adj[size_t(j)].push_back(i);
      }
    for (auto& a : adj) {
      std::sort(a.begin(), a.end());
      a.erase(std::unique(a.begin(), a.end()), a.end());
    }
    const std::vector<int> order = standin::minimum_degree(std::move(adj));
    perm.indices().v.assign(order.begin(), order.end());
  }
};

template <typename MatrixType>
class SparseLU {
 public:
  struct TransposeProxy {
    const SparseLU* lu;
    MatrixXd solve(const MatrixXd& b) const { return lu->solve_impl(b, true); }
  };

  void isSymmetric(bool sym) { symmetric_ = sym; }

  // Column ordering: minimum degree on pattern(A'A) (the COLAMD target).
  void analyzePattern(const MatrixType& a) {
    const int n = int(a.cols());
    std::vector<std::vector<int>> rows_of(size_t(a.rows()));
    for (int j = 0; j < n; ++j)
      for (auto k = a.colptr()[size_t(j)]; k < a.colptr()[size_t(j) + 1]; ++k)
        rows_of[size_t(a.rowind()[size_t(k)])].push_back(j);
    std::vector<std::vector<int>> adj(static_cast<size_t>(n));
    for (const auto& cols : rows_of)
      for (int c1 : cols)
        for (int c2 : cols)
          if (c1 != c2) adj[size_t(c1)].push_back(c2);
    for (auto& v : adj) {
      std::sort(v.begin(), v.end());
      v.erase(std::unique(v.begin(), v.end()), v.end());
    }
    q_ = standin::minimum_degree(std::move(adj));
    analyzed_ = true;
  }

  // Left-looking LU with partial pivoting on A(:, q).
  void factorize(const MatrixType& a) {
    if (!analyzed_) analyzePattern(a);
    const int n = int(a.cols());
    n_ = n;
    info_ = Success;
    lp_.assign(1, 0);
    li_.clear();
    lx_.clear();
    up_.assign(1, 0);
    ui_.clear();
    ux_.clear();
    udiag_.assign(size_t(n), 0.0);
    pinv_.assign(size_t(n), -1);
    prow_.assign(size_t(n), -1);
    std::vector<double> x(size_t(n), 0.0);
    std::vector<int> mark(size_t(n), -1), stack, pstack, reach;
    for (int k = 0; k < n; ++k) {
      const int col = q_[size_t(k)];
      // Reach: pivot steps whose L columns touch the pattern, in topological
      // order (reverse DFS finish order), plus the plain rows.
      reach.clear();
      std::vector<int> topo;
      for (auto e = a.colptr()[size_t(col)]; e < a.colptr()[size_t(col) + 1]; ++e) {
        const int r = int(a.rowind()[size_t(e)]);
        if (mark[size_t(r)] == k) continue;
        // iterative DFS from row r
        stack.assign(1, r);
        pstack.assign(1, 0);
        mark[size_t(r)] = k;
        while (!stack.empty()) {
          const int rr = stack.back();
          const int s = pinv_[size_t(rr)];
          bool pushed = false;
          if (s >= 0) {
            int& p = pstack.back();
            const int lo = lp_[size_t(s)] + p, hi = lp_[size_t(s) + 1];
            for (int t = lo; t < hi; ++t) {
              ++p;
              const int i = li_[size_t(t)];
              if (mark[size_t(i)] != k) {
                mark[size_t(i)] = k;
                stack.push_back(i);
                pstack.push_back(0);
                pushed = true;
                break;
              }
            }
          }
          if (!pushed) {
            topo.push_back(rr);
            stack.pop_back();
            pstack.pop_back();
          }
        }
      }
      std::reverse(topo.begin(), topo.end());
      for (auto e = a.colptr()[size_t(col)]; e < a.colptr()[size_t(col) + 1]; ++e)
        x[size_t(a.rowind()[size_t(e)])] += a.values()[size_t(e)];
      for (int r : topo) {
        const int s = pinv_[size_t(r)];
        if (s < 0) continue;
        const double xr = x[size_t(r)];
        if (xr == 0.0) continue;
        for (int t = lp_[size_t(s)]; t < lp_[size_t(s) + 1]; ++t)
          x[size_t(li_[size_t(t)])] -= lx_[size_t(t)] * xr;
      }
      // pivot: largest magnitude among unpivoted rows; the diagonal of the
      // permuted matrix (row col) wins ties
      int piv = -1;
      double best = -1.0;
      for (int r : topo) {
        if (pinv_[size_t(r)] >= 0) continue;
        const double v = std::abs(x[size_t(r)]);
        if (v > best || (v == best && r == col)) {
          best = v;
          piv = r;
        }
      }
      if (piv < 0 || best == 0.0 || !std::isfinite(best)) {
        info_ = NumericalIssue;
        for (int r : topo) x[size_t(r)] = 0.0;
        return;
      }
      const double pv = x[size_t(piv)];
      for (int r : topo) {
        const int s = pinv_[size_t(r)];
        if (s >= 0) {
          ui_.push_back(s);
          ux_.push_back(x[size_t(r)]);
        }
      }
      up_.push_back(int(ui_.size()));
      udiag_[size_t(k)] = pv;
      pinv_[size_t(piv)] = k;
      prow_[size_t(k)] = piv;
      for (int r : topo) {
        if (pinv_[size_t(r)] < 0) {
          li_.push_back(r);
          lx_.push_back(x[size_t(r)] / pv);
        }
        x[size_t(r)] = 0.0;
      }
      lp_.push_back(int(li_.size()));
    }
    // relabel L rows into pivot-step order
    for (auto& r : li_) r = pinv_[size_t(r)];
  }

  ComputationInfo info() const { return info_; }

  MatrixXd solve(const MatrixXd& b) const { return solve_impl(b, false); }
  TransposeProxy transpose() const { return {this}; }

 private:
  MatrixXd solve_impl(const MatrixXd& b, bool trans) const {
    const int n = n_;
    if (b.rows() != n) throw std::runtime_error("SparseLU stand-in: rhs rows");
    MatrixXd out(b.rows(), b.cols());
    std::vector<double> c(static_cast<size_t>(n));
    for (long j = 0; j < b.cols(); ++j) {
      const double* bj = b.data() + j * n;
      double* oj = out.data() + j * n;
      if (!trans) {
        for (int k = 0; k < n; ++k) c[size_t(k)] = bj[prow_[size_t(k)]];
        for (int k = 0; k < n; ++k) {  // L (unit, column-oriented)
          const double ck = c[size_t(k)];
          if (ck == 0.0) continue;
          for (int t = lp_[size_t(k)]; t < lp_[size_t(k) + 1]; ++t)
            c[size_t(li_[size_t(t)])] -= lx_[size_t(t)] * ck;
        }
        for (int k = n - 1; k >= 0; --k) {  // U (column-oriented)
          const double ck = c[size_t(k)] / udiag_[size_t(k)];
          c[size_t(k)] = ck;
          if (ck == 0.0) continue;
          for (int t = up_[size_t(k)]; t < up_[size_t(k) + 1]; ++t)
            c[size_t(ui_[size_t(t)])] -= ux_[size_t(t)] * ck;
        }
        for (int k = 0; k < n; ++k) oj[q_[size_t(k)]] = c[size_t(k)];
      } else {
        for (int k = 0; k < n; ++k) c[size_t(k)] = bj[q_[size_t(k)]];
        for (int k = 0; k < n; ++k) {  // U' (row k of U' = column k of U)
          double acc = c[size_t(k)];
          for (int t = up_[size_t(k)]; t < up_[size_t(k) + 1]; ++t)
            acc -= ux_[size_t(t)] * c[size_t(ui_[size_t(t)])];
          c[size_t(k)] = acc / udiag_[size_t(k)];
        }
        for (int k = n - 1; k >= 0; --k) {  // L' (unit upper)
          double acc = c[size_t(k)];
          for (int t = lp_[size_t(k)]; t < lp_[size_t(k) + 1]; ++t)
            acc -= lx_[size_t(t)] * c[size_t(li_[size_t(t)])];
          c[size_t(k)] = acc;
        }
        for (int k = 0; k < n; ++k) oj[prow_[size_t(k)]] = c[size_t(k)];
      }
    }
    return out;
  }

  bool symmetric_ = false, analyzed_ = false;
  int n_ = 0;
  ComputationInfo info_ = Success;
  std::vector<int> q_;            // column order: step k factors column q_[k]
  std::vector<int> pinv_, prow_;  // row -> step, step -> row
  std::vector<int> lp_, li_, up_, ui_;
  std::vector<double> lx_, ux_, udiag_;
};

}  // namespace Eigen
