// Univariate numerics of the setup path: Gauss-Legendre rules, symmetric
// banded storage + Cholesky, B-spline spaces, Gram matrices, two-scale
// (knot-insertion) matrices, and the symmetric-definite generalized
// eigendecomposition behind fast diagonalization.
//
// Restates, Eigen-free:
//   quadrature.hpp/.cpp  (/root/reference/proj/src/quadrature.cpp:14-58)
//   banded.hpp/.cpp      (/root/reference/proj/src/banded.cpp:10-77)
//   spline.hpp/.cpp      (/root/reference/proj/src/spline.cpp:11-222)
#pragma once

#include <array>
#include <vector>

#include "core.hpp"

namespace pmg {

inline constexpr int kMaxDegree = 8;  // spline.hpp:12

// ---------------------------------------------------------------- quadrature
struct QuadratureRule {
  std::vector<double> nodes;    // ascending, in (0,1)
  std::vector<double> weights;  // sum to 1
};
/// Gauss-Legendre on [0,1], cached per order (quadrature.cpp:50-58).
const QuadratureRule& gauss_legendre(int points);

// ---------------------------------------------------------------- banded
/// Lower band stored row-wise: (i,j), j<=i, i-j<=bw at data[i*(bw+1)+(i-j)]
/// (banded.hpp:9-10).
class BandedSymMatrix {
 public:
  BandedSymMatrix() = default;
  BandedSymMatrix(int dim, int bw) : dim_(dim), bw_(bw), data_(std::size_t(dim) * (bw + 1), 0.0) {}
  int dim() const { return dim_; }
  int bandwidth() const { return bw_; }
  double operator()(int i, int j) const;
  void add(int i, int j, double v);
  Dense to_dense() const;
  static BandedSymMatrix combine(double alpha, const BandedSymMatrix& A, double beta,
                                 const BandedSymMatrix& B);
  const std::vector<double>& data() const { return data_; }

 private:
  int dim_ = 0, bw_ = 0;
  std::vector<double> data_;
};

/// Banded Cholesky (banded.cpp:43-59); solve (banded.cpp:61-77).
class BandedCholesky {
 public:
  BandedCholesky() = default;
  explicit BandedCholesky(const BandedSymMatrix& a);
  int dim() const { return dim_; }
  int bandwidth() const { return bw_; }
  const std::vector<double>& factor() const { return l_; }
  void solve(const double* rhs, double* out) const;

 private:
  int dim_ = 0, bw_ = 0;
  std::vector<double> l_;
};

// ---------------------------------------------------------------- spline
enum class EndCondition { free_end, eliminated };

/// Open-uniform, maximally smooth univariate space (spline.hpp:22-58).
class UnivariateSpace {
 public:
  UnivariateSpace(int degree, int elements, EndCondition left = EndCondition::free_end,
                  EndCondition right = EndCondition::free_end);
  int degree() const { return degree_; }
  int elements() const { return elements_; }
  double mesh_size() const { return 1.0 / elements_; }
  EndCondition left() const { return left_; }
  EndCondition right() const { return right_; }
  int full_dimension() const { return elements_ + degree_; }
  int dimension() const {
    return full_dimension() - (left_ == EndCondition::eliminated ? 1 : 0) -
           (right_ == EndCondition::eliminated ? 1 : 0);
  }
  int first_active() const { return left_ == EndCondition::eliminated ? 1 : 0; }
  int to_reduced(int full_index) const {
    int r = full_index - first_active();
    return (r >= 0 && r < dimension()) ? r : -1;
  }
  std::vector<double> knots() const;
  bool operator==(const UnivariateSpace& o) const {
    return degree_ == o.degree_ && elements_ == o.elements_ && left_ == o.left_ && right_ == o.right_;
  }

 private:
  int degree_, elements_;
  EndCondition left_, right_;
};

struct BasisEval {
  int first_index = 0;
  std::array<double, kMaxDegree + 1> values{};
};

/// Cox-de Boor values / first derivatives at x in [0,1] (spline.cpp:26-82).
BasisEval eval_basis(const UnivariateSpace& space, double x, int deriv = 0);

/// Gram matrices over the eliminated basis (spline.cpp:86-110,141-145).
BandedSymMatrix univariate_mass(const UnivariateSpace& space);
BandedSymMatrix univariate_stiffness(const UnivariateSpace& space);

/// Rectangular two-scale matrix with contiguous row support (spline.hpp:76-85,
/// spline.cpp:172-204).
struct TwoScaleMatrix {
  int fine_dim = 0;
  int coarse_dim = 0;
  std::vector<int> row_start;
  std::vector<std::vector<double>> row_vals;
  Dense to_dense() const;
};
TwoScaleMatrix two_scale_matrix(const UnivariateSpace& coarse);

/// Boehm single-knot insertion on a refinement matrix (spline.cpp:115-137).
void insert_knot(std::vector<double>& knots, int degree, double u, Dense& refine);

/// K v = lambda M v with V^T M V = I, eigenvalues ascending, negatives within
/// 1e-9 relative clamped to 0 (spline.cpp:206-222).  Eigen's
/// GeneralizedSelfAdjointEigenSolver(Ax_lBx) is restated as Cholesky of M,
/// C = L^-1 K L^-T, cyclic Jacobi on C, V = L^-T Q.
struct GenEigDecomposition {
  std::vector<double> eigenvalues;
  Dense eigenvectors;  // columns
};
GenEigDecomposition gen_eig(const Dense& K, const Dense& M);

/// Dense Cholesky A = L L^T (lower, column-major); throws DefinitenessError.
Dense dense_cholesky(const Dense& A);
/// Solve L L^T x = b in place with the factor from dense_cholesky.
void dense_cholesky_solve(const Dense& L, double* b);

}  // namespace pmg
