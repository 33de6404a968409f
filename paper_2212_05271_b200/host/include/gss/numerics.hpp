// gss/numerics.hpp (B200 build) -- minimal dense complex matrix / vector value types standing in for the
// Eigen::MatrixXcd / VectorXcd members of the reference's public structs (cacgmm.hpp:27, beamform.hpp:22-29).
// Same element access ((r,c), rows(), cols(), size()); storage is row-major, which is what the C ABI moves.
// The Hermitian helpers of numerics.hpp:28-152 have no host implementation here: they run inside the
// device kernels (csrc/linalg.cuh).
#pragma once

#include <vector>

#include "common.hpp"

namespace gss::numerics {

constexpr double kDefaultRegEps = 1e-10;          // numerics.hpp:28
constexpr double kEigenvalueFloorRatio = 1e-10;   // numerics.hpp:29

class CMatrix {
 public:
  CMatrix() = default;
  CMatrix(int rows, int cols) : r_(rows), c_(cols), v_(static_cast<size_t>(rows) * cols) {}
  static CMatrix Identity(int n, int m) {
    CMatrix a(n, m);
    for (int i = 0; i < n && i < m; ++i) a(i, i) = 1.0;
    return a;
  }
  int rows() const { return r_; }
  int cols() const { return c_; }
  cdouble& operator()(int r, int c) { return v_[static_cast<size_t>(r) * c_ + c]; }
  const cdouble& operator()(int r, int c) const { return v_[static_cast<size_t>(r) * c_ + c]; }
  cdouble* data() { return v_.data(); }
  const cdouble* data() const { return v_.data(); }

 private:
  int r_ = 0, c_ = 0;
  std::vector<cdouble> v_;
};

using CVector = std::vector<cdouble>;

}  // namespace gss::numerics
