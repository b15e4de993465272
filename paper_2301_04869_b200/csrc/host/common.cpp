#include "common.hpp"

#include <algorithm>

namespace bipm {

idx Csr::find(idx i, idx j) const {
  auto b = ind.begin() + ptr[size_t(i)], e = ind.begin() + ptr[size_t(i) + 1];
  auto it = std::lower_bound(b, e, j);
  return (it != e && *it == j) ? idx(it - ind.begin()) : -1;
}

Csr Csr::pattern(idx rows, idx cols, std::vector<std::pair<idx, idx>> coords) {
  std::sort(coords.begin(), coords.end());
  coords.erase(std::unique(coords.begin(), coords.end()), coords.end());
  Csr p;
  p.rows = rows;
  p.cols = cols;
  p.ptr.assign(size_t(rows) + 1, 0);
  p.ind.reserve(coords.size());
  for (const auto& [i, j] : coords) {
    if (i < 0 || i >= rows || j < 0 || j >= cols)
      throw Error(kInvalidArgument, "pattern coordinate out of range");
    ++p.ptr[size_t(i) + 1];
    p.ind.push_back(j);
  }
  for (idx i = 0; i < rows; ++i) p.ptr[size_t(i) + 1] += p.ptr[size_t(i)];
  return p;
}

Csr Csr::assemble(idx rows, idx cols, std::vector<std::pair<std::pair<idx, idx>, double>> t) {
  // stable: duplicates keep insertion order and are summed left to right
  std::stable_sort(t.begin(), t.end(),
                   [](const auto& a, const auto& b) { return a.first < b.first; });
  Csr m;
  m.rows = rows;
  m.cols = cols;
  m.ptr.assign(size_t(rows) + 1, 0);
  for (size_t k = 0; k < t.size(); ++k) {
    if (k > 0 && t[k].first == t[k - 1].first) {
      m.val.back() += t[k].second;
      continue;
    }
    ++m.ptr[size_t(t[k].first.first) + 1];
    m.ind.push_back(t[k].first.second);
    m.val.push_back(t[k].second);
  }
  for (idx i = 0; i < rows; ++i) m.ptr[size_t(i) + 1] += m.ptr[size_t(i)];
  return m;
}

Csr Csr::transpose_pattern() const {
  Csr t;
  t.rows = cols;
  t.cols = rows;
  t.ptr.assign(size_t(cols) + 1, 0);
  for (idx j : ind) ++t.ptr[size_t(j) + 1];
  for (idx j = 0; j < cols; ++j) t.ptr[size_t(j) + 1] += t.ptr[size_t(j)];
  t.ind.resize(ind.size());
  t.val.resize(ind.size());
  std::vector<idx> fill(t.ptr.begin(), t.ptr.end() - 1);
  for (idx i = 0; i < rows; ++i)
    for (idx k = ptr[size_t(i)]; k < ptr[size_t(i) + 1]; ++k) {
      const idx pos = fill[size_t(ind[size_t(k)])]++;
      t.ind[size_t(pos)] = i;
      t.val[size_t(pos)] = double(k);
    }
  return t;
}

}  // namespace bipm
