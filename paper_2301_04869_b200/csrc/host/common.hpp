// Shared host-side types for the B200 reduced-KKT solver.
//
// Layout convention (same as the reference boundary,
// proj/core/include/blockipm/types.hpp:56-78): per-scenario arrays are stored
// scenario-major, i.e. scenario b's `len` values are the contiguous range
// [b*len, (b+1)*len).  Patterns are shared int32 CSR.
#pragma once

#include <cstdint>
#include <limits>
#include <stdexcept>
#include <string>
#include <vector>

namespace bipm {

using idx = std::int32_t;
inline constexpr double kInf = std::numeric_limits<double>::infinity();

// Status codes crossing the C-ABI (include/bipm_gpu.h).  They map one-to-one
// onto the reference's exception types.
enum Status : int {
  kOk = 0,
  kSingularBlock = 1,   // SingularBlockError (types.hpp:99-103)
  kNonFinite = 2,       // NonFiniteError (types.hpp:105-109)
  kNotPd = 3,           // dense factor not positive definite (kkt.cpp:970-971)
  kCudaError = 4,
  kInvalidArgument = 5,  // DimensionError / std::invalid_argument
  kNonInterior = 6,      // NonInteriorError (kkt.hpp:31-33)
  kLinearSolve = 7,      // LinearSolveError (kkt.hpp:34-36)
  kParseError = 8,       // opf::ParseError
  kUnsupported = 9,      // a path the GPU engine does not implement (augmented fallback)
};

struct Error : std::runtime_error {
  int code;
  idx block;  // offending scenario (global index) or -1
  Error(int c, const std::string& what, idx b = -1) : std::runtime_error(what), code(c), block(b) {}
};

// Compressed-row pattern with optional values.
struct Csr {
  idx rows = 0, cols = 0;
  std::vector<idx> ptr{0};
  std::vector<idx> ind;
  std::vector<double> val;  // empty for a pure pattern

  idx nnz() const { return idx(ind.size()); }
  idx find(idx i, idx j) const;  // slot of (i, j) or -1
  // Sorted-unique pattern from coordinates (duplicates dropped).
  static Csr pattern(idx rows, idx cols, std::vector<std::pair<idx, idx>> coords);
  // Values from (row, col, value) entries; duplicates accumulate in input order.
  static Csr assemble(idx rows, idx cols, std::vector<std::pair<std::pair<idx, idx>, double>> t);
  Csr transpose_pattern() const;  // pattern of A' with `val` = source slot index as double
};

}  // namespace bipm
