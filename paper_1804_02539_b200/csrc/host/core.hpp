// Shared host-side core types for the hierarchy setup library.
//
// Error classes mirror /root/reference/proj/include/patchmg/errors.hpp:9-56 one
// for one (same names, same meaning), so the C ABI can map them onto the same
// status codes the reference's CLI maps onto exit codes (harness.cpp:573-581).
// The dense matrix is a minimal column-major container standing in for the
// Eigen::MatrixXd the reference uses in its setup code.
#pragma once

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace pmg {

struct Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ConfigError : Error { using Error::Error; };
struct DomainError : Error { using Error::Error; };
struct NonMatchingError : Error { using Error::Error; };
struct NonManifoldError : Error { using Error::Error; };
struct SingularGeometryError : Error { using Error::Error; };
struct DecompositionError : Error { using Error::Error; };
struct DefinitenessError : Error { using Error::Error; };
struct DivergenceError : Error { using Error::Error; };
struct TransportError : Error { using Error::Error; };

/// Column-major dense matrix (rows x cols), value-initialised to zero.
struct Dense {
  int rows = 0, cols = 0;
  std::vector<double> a;
  Dense() = default;
  Dense(int r, int c) : rows(r), cols(c), a(std::size_t(r) * std::size_t(c), 0.0) {}
  double& operator()(int i, int j) { return a[std::size_t(j) * rows + i]; }
  double operator()(int i, int j) const { return a[std::size_t(j) * rows + i]; }
  double* data() { return a.data(); }
  const double* data() const { return a.data(); }
  static Dense identity(int n) {
    Dense d(n, n);
    for (int i = 0; i < n; ++i) d(i, i) = 1.0;
    return d;
  }
};

}  // namespace pmg
