// Univariate numerics of the setup path (see numerics.hpp for the reference map).
#include "numerics.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <mutex>

namespace pmg {

// ============================================================ quadrature
namespace {

// P_n and P_n' by the three-term recurrence (quadrature.cpp:14-23).
std::pair<double, double> legendre(int n, double x) {
  double p0 = 1.0, p1 = x;
  for (int k = 2; k <= n; ++k) {
    double p2 = ((2 * k - 1) * x * p1 - (k - 1) * p0) / k;
    p0 = p1;
    p1 = p2;
  }
  double dp = n * (x * p1 - p0) / (x * x - 1.0);
  return {p1, dp};
}

// Newton from a Chebyshev-type guess, mapped to [0,1] (quadrature.cpp:25-46).
QuadratureRule compute_rule(int q) {
  QuadratureRule rule;
  rule.nodes.resize(q);
  rule.weights.resize(q);
  for (int i = 0; i < q; ++i) {
    double x = std::cos(M_PI * (i + 0.75) / (q + 0.5));
    for (int it = 0; it < 100; ++it) {
      auto [p, dp] = legendre(q, x);
      double dx = p / dp;
      x -= dx;
      if (std::abs(dx) < 1e-15) break;
    }
    auto [p, dp] = legendre(q, x);
    (void)p;
    double w = 2.0 / ((1.0 - x * x) * dp * dp);
    rule.nodes[q - 1 - i] = 0.5 * (x + 1.0);
    rule.weights[q - 1 - i] = 0.5 * w;
  }
  return rule;
}

}  // namespace

const QuadratureRule& gauss_legendre(int points) {
  if (points < 1 || points > 64) throw DomainError("gauss_legendre: order out of range");
  static std::map<int, QuadratureRule> cache;
  static std::mutex mtx;
  std::lock_guard<std::mutex> lock(mtx);
  auto it = cache.find(points);
  if (it == cache.end()) it = cache.emplace(points, compute_rule(points)).first;
  return it->second;
}

// ============================================================ banded
double BandedSymMatrix::operator()(int i, int j) const {
  if (j > i) std::swap(i, j);
  if (i - j > bw_) return 0.0;
  return data_[std::size_t(i) * (bw_ + 1) + (i - j)];
}

void BandedSymMatrix::add(int i, int j, double v) {
  if (j > i) std::swap(i, j);
  data_[std::size_t(i) * (bw_ + 1) + (i - j)] += v;
}

Dense BandedSymMatrix::to_dense() const {
  Dense m(dim_, dim_);
  for (int i = 0; i < dim_; ++i)
    for (int j = std::max(0, i - bw_); j <= i; ++j) m(i, j) = m(j, i) = (*this)(i, j);
  return m;
}

// banded.cpp:31-41
BandedSymMatrix BandedSymMatrix::combine(double alpha, const BandedSymMatrix& A, double beta,
                                         const BandedSymMatrix& B) {
  if (A.dim() != B.dim()) throw DomainError("BandedSymMatrix::combine: dimension mismatch");
  BandedSymMatrix out(A.dim(), std::max(A.bandwidth(), B.bandwidth()));
  for (int i = 0; i < out.dim(); ++i)
    for (int j = std::max(0, i - out.bw_); j <= i; ++j) {
      double v = alpha * A(i, j) + beta * B(i, j);
      if (v != 0.0) out.add(i, j, v);
    }
  return out;
}

// banded.cpp:43-59
BandedCholesky::BandedCholesky(const BandedSymMatrix& a)
    : dim_(a.dim()), bw_(a.bandwidth()), l_(std::size_t(a.dim()) * (a.bandwidth() + 1), 0.0) {
  const int w = bw_ + 1;
  for (int i = 0; i < dim_; ++i) {
    for (int j = std::max(0, i - bw_); j <= i; ++j) {
      double sum = a(i, j);
      int k0 = std::max({0, i - bw_, j - bw_});
      for (int k = k0; k < j; ++k) sum -= l_[std::size_t(i) * w + (i - k)] * l_[std::size_t(j) * w + (j - k)];
      if (i == j) {
        if (sum <= 0.0) throw DefinitenessError("banded Cholesky: non-positive pivot");
        l_[std::size_t(i) * w] = std::sqrt(sum);
      } else {
        l_[std::size_t(i) * w + (i - j)] = sum / l_[std::size_t(j) * w];
      }
    }
  }
}

// banded.cpp:61-77
void BandedCholesky::solve(const double* rhs, double* y) const {
  const int w = bw_ + 1;
  for (int i = 0; i < dim_; ++i) {
    double s = rhs[i];
    for (int k = std::max(0, i - bw_); k < i; ++k) s -= l_[std::size_t(i) * w + (i - k)] * y[k];
    y[i] = s / l_[std::size_t(i) * w];
  }
  for (int i = dim_ - 1; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < std::min(dim_, i + bw_ + 1); ++k) s -= l_[std::size_t(k) * w + (k - i)] * y[k];
    y[i] = s / l_[std::size_t(i) * w];
  }
}

// ============================================================ spline
UnivariateSpace::UnivariateSpace(int degree, int elements, EndCondition left, EndCondition right)
    : degree_(degree), elements_(elements), left_(left), right_(right) {
  if (degree < 1 || degree > kMaxDegree) throw DomainError("UnivariateSpace: degree out of range");
  if (elements < 1) throw DomainError("UnivariateSpace: need at least one element");
}

std::vector<double> UnivariateSpace::knots() const {
  std::vector<double> t;
  t.reserve(2 * (degree_ + 1) + elements_ - 1);
  for (int i = 0; i <= degree_; ++i) t.push_back(0.0);
  for (int e = 1; e < elements_; ++e) t.push_back(double(e) / elements_);
  for (int i = 0; i <= degree_; ++i) t.push_back(1.0);
  return t;
}

// Triangular Cox-de Boor with clamped knot lookup (spline.cpp:26-82).
BasisEval eval_basis(const UnivariateSpace& space, double x, int deriv) {
  if (!(x >= 0.0 && x <= 1.0)) throw DomainError("eval_basis: x outside [0,1]");
  if (deriv < 0 || deriv > 1) throw DomainError("eval_basis: deriv must be 0 or 1");
  const int p = space.degree();
  const int n = space.elements();
  const int e = std::min(int(x * n), n - 1);
  auto knot = [&](int i) { return std::clamp(double(i - p) / n, 0.0, 1.0); };
  const int k = e + p;

  std::array<double, kMaxDegree + 1> N{}, left{}, right{};
  N[0] = 1.0;
  const int top = deriv == 1 ? p - 1 : p;
  for (int deg = 1; deg <= top; ++deg) {
    left[deg] = x - knot(k + 1 - deg);
    right[deg] = knot(k + deg) - x;
    double saved = 0.0;
    for (int r = 0; r < deg; ++r) {
      double denom = right[r + 1] + left[deg - r];
      double tmp = denom != 0.0 ? N[r] / denom : 0.0;
      N[r] = saved + right[r + 1] * tmp;
      saved = left[deg - r] * tmp;
    }
    N[deg] = saved;
  }

  BasisEval out;
  out.first_index = e;
  out.values.fill(0.0);
  if (deriv == 0) {
    for (int j = 0; j <= p; ++j) out.values[j] = N[j];
    return out;
  }
  for (int j = 0; j <= p; ++j) {
    const int i = k - p + j;
    double a = 0.0, b = 0.0;
    if (j >= 1) {
      double denom = knot(i + p) - knot(i);
      if (denom != 0.0) a = N[j - 1] / denom;
    }
    if (j <= p - 1) {
      double denom = knot(i + p + 1) - knot(i + 1);
      if (denom != 0.0) b = N[j] / denom;
    }
    out.values[j] = p * (a - b);
  }
  return out;
}

namespace {

// spline.cpp:86-110
BandedSymMatrix univariate_gram(const UnivariateSpace& space, int deriv) {
  const int p = space.degree();
  const int n = space.elements();
  const auto& rule = gauss_legendre(p + 1);
  BandedSymMatrix m(space.dimension(), p);
  const double h = space.mesh_size();
  for (int e = 0; e < n; ++e) {
    for (std::size_t q = 0; q < rule.nodes.size(); ++q) {
      double x = (e + rule.nodes[q]) * h;
      BasisEval be = eval_basis(space, x, deriv);
      double w = rule.weights[q] * h;
      for (int a = 0; a <= p; ++a) {
        int ia = space.to_reduced(be.first_index + a);
        if (ia < 0) continue;
        for (int b = 0; b <= a; ++b) {
          int ib = space.to_reduced(be.first_index + b);
          if (ib < 0) continue;
          m.add(ia, ib, w * be.values[a] * be.values[b]);
        }
      }
    }
  }
  return m;
}

}  // namespace

BandedSymMatrix univariate_mass(const UnivariateSpace& space) { return univariate_gram(space, 0); }
BandedSymMatrix univariate_stiffness(const UnivariateSpace& space) { return univariate_gram(space, 1); }

// spline.cpp:115-137
void insert_knot(std::vector<double>& knots, int p, double u, Dense& refine) {
  const int k = int(std::upper_bound(knots.begin(), knots.end(), u) - knots.begin()) - 1;
  const int rows = refine.rows;
  Dense out(rows + 1, refine.cols);
  for (int i = 0; i <= rows; ++i) {
    double alpha;
    if (i <= k - p)
      alpha = 1.0;
    else if (i > k)
      alpha = 0.0;
    else
      alpha = (u - knots[i]) / (knots[i + p] - knots[i]);
    for (int c = 0; c < refine.cols; ++c) {
      if (alpha == 1.0)
        out(i, c) = refine(i, c);
      else if (alpha == 0.0)
        out(i, c) = refine(i - 1, c);
      else
        out(i, c) = alpha * refine(i, c) + (1.0 - alpha) * refine(i - 1, c);
    }
  }
  knots.insert(std::upper_bound(knots.begin(), knots.end(), u), u);
  refine = std::move(out);
}

Dense TwoScaleMatrix::to_dense() const {
  Dense m(fine_dim, coarse_dim);
  for (int i = 0; i < fine_dim; ++i)
    for (std::size_t k = 0; k < row_vals[i].size(); ++k) m(i, row_start[i] + int(k)) = row_vals[i][k];
  return m;
}

// spline.cpp:172-204
TwoScaleMatrix two_scale_matrix(const UnivariateSpace& coarse) {
  const int p = coarse.degree();
  const int n = coarse.elements();
  std::vector<double> knots = coarse.knots();
  Dense refine = Dense::identity(coarse.full_dimension());
  for (int e = 0; e < n; ++e) insert_knot(knots, p, (e + 0.5) / n, refine);

  UnivariateSpace fine(p, 2 * n, coarse.left(), coarse.right());
  TwoScaleMatrix out;
  out.fine_dim = fine.dimension();
  out.coarse_dim = coarse.dimension();
  out.row_start.assign(out.fine_dim, 0);
  out.row_vals.resize(out.fine_dim);
  const int fshift = fine.first_active();
  const int cshift = coarse.first_active();
  for (int i = 0; i < out.fine_dim; ++i) {
    int lo = -1, hi = -1;
    for (int j = 0; j < out.coarse_dim; ++j) {
      if (refine(i + fshift, j + cshift) != 0.0) {
        if (lo < 0) lo = j;
        hi = j;
      }
    }
    if (lo < 0) continue;
    out.row_start[i] = lo;
    out.row_vals[i].resize(hi - lo + 1);
    for (int j = lo; j <= hi; ++j) out.row_vals[i][j - lo] = refine(i + fshift, j + cshift);
  }
  return out;
}

// ============================================================ dense SPD helpers
Dense dense_cholesky(const Dense& A) {
  const int n = A.rows;
  Dense L(n, n);
  for (int j = 0; j < n; ++j) {
    double d = A(j, j);
    for (int k = 0; k < j; ++k) d -= L(j, k) * L(j, k);
    if (!(d > 0.0)) throw DefinitenessError("dense Cholesky: matrix is not positive definite");
    const double ljj = std::sqrt(d);
    L(j, j) = ljj;
    for (int i = j + 1; i < n; ++i) {
      double s = A(i, j);
      for (int k = 0; k < j; ++k) s -= L(i, k) * L(j, k);
      L(i, j) = s / ljj;
    }
  }
  return L;
}

void dense_cholesky_solve(const Dense& L, double* b) {
  const int n = L.rows;
  for (int i = 0; i < n; ++i) {  // L y = b
    double s = b[i];
    for (int k = 0; k < i; ++k) s -= L(i, k) * b[k];
    b[i] = s / L(i, i);
  }
  for (int i = n - 1; i >= 0; --i) {  // L^T x = y
    double s = b[i];
    for (int k = i + 1; k < n; ++k) s -= L(k, i) * b[k];
    b[i] = s / L(i, i);
  }
}

namespace {

// Cyclic Jacobi on a symmetric matrix (column-major, overwritten).  Returns
// the eigenvector matrix; eigenvalues are left on the diagonal of A.
Dense jacobi_eigen(Dense& A) {
  const int n = A.rows;
  Dense V = Dense::identity(n);
  double frob = 0.0;
  for (double v : A.a) frob += v * v;
  if (frob == 0.0) return V;
  for (int sweep = 0; sweep < 100; ++sweep) {
    double off = 0.0;
    for (int q = 1; q < n; ++q)
      for (int p = 0; p < q; ++p) off += A(p, q) * A(p, q);
    if (off <= 1e-34 * frob) break;
    for (int p = 0; p < n - 1; ++p) {
      for (int q = p + 1; q < n; ++q) {
        const double apq = A(p, q);
        if (apq == 0.0) continue;
        const double app = A(p, p), aqq = A(q, q);
        if (sweep > 3 && std::abs(apq) < 1e-18 * std::abs(app) && std::abs(apq) < 1e-18 * std::abs(aqq)) {
          A(p, q) = A(q, p) = 0.0;
          continue;
        }
        const double theta = (aqq - app) / (2.0 * apq);
        const double t = (theta >= 0.0 ? 1.0 : -1.0) / (std::abs(theta) + std::sqrt(theta * theta + 1.0));
        const double c = 1.0 / std::sqrt(t * t + 1.0);
        const double s = t * c;
        double* cp = &A(0, p);
        double* cq = &A(0, q);
        for (int k = 0; k < n; ++k) {  // columns: A J
          const double akp = cp[k], akq = cq[k];
          cp[k] = c * akp - s * akq;
          cq[k] = s * akp + c * akq;
        }
        for (int k = 0; k < n; ++k) {  // rows: J^T (A J)
          const double apk = A(p, k), aqk = A(q, k);
          A(p, k) = c * apk - s * aqk;
          A(q, k) = s * apk + c * aqk;
        }
        A(p, q) = A(q, p) = 0.0;
        double* vp = &V(0, p);
        double* vq = &V(0, q);
        for (int k = 0; k < n; ++k) {
          const double a0 = vp[k], a1 = vq[k];
          vp[k] = c * a0 - s * a1;
          vq[k] = s * a0 + c * a1;
        }
      }
    }
  }
  return V;
}

}  // namespace

// spline.cpp:206-222
GenEigDecomposition gen_eig(const Dense& K, const Dense& M) {
  if (K.rows != K.cols || M.rows != M.cols || K.rows != M.rows) throw DomainError("gen_eig: shape mismatch");
  const int n = K.rows;
  Dense L;
  try {
    L = dense_cholesky(M);
  } catch (const DefinitenessError&) {
    throw DefinitenessError("gen_eig: M is not positive definite");
  }
  // Y = L^-1 K (forward substitution on every column)
  Dense Y = K;
  for (int c = 0; c < n; ++c)
    for (int i = 0; i < n; ++i) {
      double s = Y(i, c);
      for (int k = 0; k < i; ++k) s -= L(i, k) * Y(k, c);
      Y(i, c) = s / L(i, i);
    }
  // C = L^-1 Y^T  (= L^-1 K L^-T)
  Dense C(n, n);
  for (int c = 0; c < n; ++c)
    for (int i = 0; i < n; ++i) {
      double s = Y(c, i);
      for (int k = 0; k < i; ++k) s -= L(i, k) * C(k, c);
      C(i, c) = s / L(i, i);
    }
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < i; ++j) {
      const double v = 0.5 * (C(i, j) + C(j, i));
      C(i, j) = C(j, i) = v;
    }
  Dense Q = jacobi_eigen(C);
  std::vector<int> order(n);
  for (int i = 0; i < n; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return C(a, a) < C(b, b); });

  GenEigDecomposition out;
  out.eigenvalues.resize(n);
  out.eigenvectors = Dense(n, n);
  for (int j = 0; j < n; ++j) {
    out.eigenvalues[j] = C(order[j], order[j]);
    // V = L^-T q  (back substitution)
    double* v = &out.eigenvectors(0, j);
    for (int i = 0; i < n; ++i) v[i] = Q(i, order[j]);
    for (int i = n - 1; i >= 0; --i) {
      double s = v[i];
      for (int k = i + 1; k < n; ++k) s -= L(k, i) * v[k];
      v[i] = s / L(i, i);
    }
  }
  const double top = n > 0 ? std::abs(out.eigenvalues[n - 1]) : 0.0;
  for (int i = 0; i < n; ++i) {
    if (out.eigenvalues[i] < -1e-9 * top)
      throw DecompositionError("gen_eig: K has a significantly negative eigenvalue");
    if (out.eigenvalues[i] < 0.0) out.eigenvalues[i] = 0.0;
  }
  return out;
}

}  // namespace pmg
