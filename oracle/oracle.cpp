// CPU oracle of the PCG + V-cycle solve path.  TEST INFRASTRUCTURE ONLY --
// see oracle.h for the reference map and the usage restriction.
//
// Arithmetic follows the reference loops in order (the reference's Release
// build has no FMA contraction; this file is compiled with
// -ffp-contract=off).  Eigen's blocked GEMM/dot reductions are restated as
// ascending-index sums, so the oracle agrees with the reference to rounding
// (tested identities at 1e-12..1e-13), not bitwise.
#include "oracle.h"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <functional>
#include <map>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

namespace oracle {

using Vec = std::vector<double>;

struct ConfigError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DomainError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DefinitenessError : std::runtime_error { using std::runtime_error::runtime_error; };
struct DivergenceError : std::runtime_error { using std::runtime_error::runtime_error; };
struct TransportError : std::runtime_error { using std::runtime_error::runtime_error; };

// ---------------------------------------------------------------- hierarchy view
struct Level {
  int n = 0, ext = 0;
  std::int64_t S = 0;  // lattice entries per patch
  std::int64_t N = 0;  // global dofs
  const std::int32_t* l2g = nullptr;
  const pmg_level_desc* desc = nullptr;
  std::vector<std::int32_t> rep_off, rep_patch, rep_local;  // DofMapper reps (topology.cpp:348-364)
  std::int32_t owner_patch(std::int32_t g) const { return rep_patch[rep_off[g]]; }
};

struct Hier {
  int d = 0, p = 0, K = 0, O = 0;
  pmg_cycle_params prm{};
  std::vector<Level> lv;
  int n0 = 0;
  const double* L0 = nullptr;
  // coarse_mode 1: the explicit inverse L^-T L^-1 applied as a GEMV, a
  // second exact coarse solver with different rounding (measures the
  // conditioning limit kappa(A_0) eps of any coarse-solve pairing)
  int coarse_mode = 0;
  std::vector<double> Ainv;
  int finest() const { return int(lv.size()) - 1; }
};

void build_view(const pmg_hierarchy_desc* D, Hier& H) {
  H.d = D->dim;
  H.p = D->degree;
  H.K = D->num_patches;
  H.O = 1;
  for (int a = 0; a < H.d; ++a) H.O *= 2 * H.p + 1;
  H.prm = D->params;
  H.n0 = D->coarse_n;
  H.L0 = D->coarse_L;
  H.lv.resize(D->num_levels);
  for (int l = 0; l < D->num_levels; ++l) {
    const pmg_level_desc& ld = D->levels[l];
    // a PMG_BAND_KRONECKER level still carries the host-assembled band: the
    // checker applies the assembled operator, as the reference does
    if ((ld.band_format != PMG_BAND_TENSOR && ld.band_format != PMG_BAND_KRONECKER) || !ld.band)
      throw ConfigError("oracle: needs host-assembled tensor bands (use a host-assembled hierarchy)");
    Level& L = H.lv[l];
    L.desc = &ld;
    L.n = ld.elements;
    L.ext = ld.elements + H.p;
    L.S = 1;
    for (int a = 0; a < H.d; ++a) L.S *= L.ext;
    L.N = ld.num_dofs;
    L.l2g = ld.l2g;
    L.rep_off.assign(std::size_t(L.N) + 1, 0);
    for (std::int64_t i = 0; i < L.S * H.K; ++i)
      if (L.l2g[i] >= 0) L.rep_off[L.l2g[i] + 1]++;
    for (std::int64_t g = 0; g < L.N; ++g) L.rep_off[g + 1] += L.rep_off[g];
    L.rep_patch.resize(L.rep_off.back());
    L.rep_local.resize(L.rep_off.back());
    std::vector<std::int32_t> cur(L.rep_off.begin(), L.rep_off.end() - 1);
    for (int k = 0; k < H.K; ++k)
      for (std::int64_t f = 0; f < L.S; ++f) {
        const std::int32_t g = L.l2g[k * L.S + f];
        if (g < 0) continue;
        L.rep_patch[cur[g]] = k;
        L.rep_local[cur[g]] = std::int32_t(f);
        cur[g]++;
      }
  }
}

// ---------------------------------------------------------------- operator
// PatchOperator::apply_add (assembly.cpp:12-18): the CSR row holds the
// tensor-band columns in lexicographic order, axis 0 fastest.
void patch_apply_add(const Hier& H, const Level& L, int k, const double* x, double* y) {
  const pmg_level_desc& ld = *L.desc;
  if (ld.band_format == PMG_BAND_CSR) {
    const std::int64_t* rp = ld.csr_row_ptr[k];
    const std::int32_t* cols = ld.csr_cols[k];
    const double* vals = ld.csr_vals[k];
    for (std::int64_t r = 0; r < L.S; ++r) {
      double acc = 0.0;
      for (std::int64_t q = rp[r]; q < rp[r + 1]; ++q) acc += vals[q] * x[cols[q]];
      y[r] += acc;
    }
    return;
  }
  const double* band = ld.band + std::size_t(k) * H.O * L.S;
  const int d = H.d, p = H.p, ext = L.ext, w = 2 * p + 1;
  int idx[3] = {0, 0, 0};
  for (std::int64_t r = 0; r < L.S; ++r) {
    double acc = 0.0;
    int lo[3] = {0, 0, 0}, hi[3] = {0, 0, 0};
    for (int a = 0; a < d; ++a) {
      lo[a] = std::max(0, idx[a] - p);
      hi[a] = std::min(ext - 1, idx[a] + p);
    }
    int j[3] = {lo[0], lo[1], lo[2]};
    for (;;) {
      std::int64_t c = 0;
      int o = 0;
      for (int a = d - 1; a >= 0; --a) {
        c = c * ext + j[a];
        o = o * w + (j[a] - idx[a] + p);
      }
      acc += band[std::size_t(o) * L.S + r] * x[c];
      int a = 0;
      for (; a < d; ++a) {
        if (++j[a] <= hi[a]) break;
        j[a] = lo[a];
      }
      if (a == d) break;
    }
    y[r] += acc;
    for (int a = 0; a < d; ++a) {
      if (++idx[a] < ext) break;
      idx[a] = 0;
    }
  }
}

// MultiPatchOperator::apply (assembly.cpp:265-280)
Vec op_apply(const Hier& H, int level, const Vec& x) {
  const Level& L = H.lv[level];
  Vec y(std::size_t(L.N), 0.0), xl, yl;
  for (int k = 0; k < H.K; ++k) {
    const std::int32_t* l2g = L.l2g + k * L.S;
    xl.assign(std::size_t(L.S), 0.0);
    yl.assign(std::size_t(L.S), 0.0);
    for (std::int64_t f = 0; f < L.S; ++f)
      if (l2g[f] >= 0) xl[f] = x[l2g[f]];
    patch_apply_add(H, L, k, xl.data(), yl.data());
    for (std::int64_t f = 0; f < L.S; ++f)
      if (l2g[f] >= 0) y[l2g[f]] += yl[f];
  }
  return y;
}

// ---------------------------------------------------------------- tensor kernels
void axis_split(const std::vector<int>& dims, int axis, std::int64_t& inner, std::int64_t& outer) {
  inner = outer = 1;
  for (int a = 0; a < axis; ++a) inner *= dims[a];
  for (std::size_t a = axis + 1; a < dims.size(); ++a) outer *= dims[a];
}

// apply_along_axis with a dense column-major m x m matrix (tensor.cpp:18-33):
// y_o = x_o M^T, summed over the contracted index in ascending order.
Vec dense_along(const double* M, int m, const Vec& x, const std::vector<int>& dims, int axis, bool transpose) {
  std::int64_t inner, outer;
  axis_split(dims, axis, inner, outer);
  Vec y(x.size(), 0.0);
  for (std::int64_t o = 0; o < outer; ++o) {
    const double* xo = x.data() + o * inner * m;
    double* yo = y.data() + o * inner * m;
    for (int i = 0; i < m; ++i) {
      double* yrow = yo + std::int64_t(i) * inner;
      for (int k = 0; k < m; ++k) {
        // non-transposed: Y(t,i) = sum_k X(t,k) M(i,k); transposed: sum_k X(t,k) M(k,i)
        const double v = transpose ? M[std::size_t(i) * m + k] : M[std::size_t(k) * m + i];
        const double* xrow = xo + std::int64_t(k) * inner;
        for (std::int64_t t = 0; t < inner; ++t) yrow[t] += v * xrow[t];
      }
    }
  }
  return y;
}

// two-scale apply_along_axis / _transpose (tensor.cpp:52-102)
Vec ts_along(const Level& Lf, const Vec& x, const std::vector<int>& dims, int axis, bool transpose) {
  const pmg_level_desc& ld = *Lf.desc;
  std::int64_t inner, outer;
  axis_split(dims, axis, inner, outer);
  const int m = dims[axis];
  const int r = transpose ? ld.ts_coarse_dim : ld.ts_fine_dim;
  if (m != (transpose ? ld.ts_fine_dim : ld.ts_coarse_dim)) throw DomainError("apply_along_axis: extent mismatch");
  Vec y(std::size_t(inner * r * outer), 0.0);
  for (std::int64_t o = 0; o < outer; ++o) {
    const double* xin = x.data() + o * inner * m;
    double* yout = y.data() + o * inner * r;
    if (!transpose) {
      for (int i = 0; i < r; ++i) {
        double* yrow = yout + std::int64_t(i) * inner;
        const double* vals = ld.ts_vals + ld.ts_row_off[i];
        for (int k = 0; k < ld.ts_row_len[i]; ++k) {
          const double v = vals[k];
          const double* xrow = xin + std::int64_t(ld.ts_row_start[i] + k) * inner;
          for (std::int64_t t = 0; t < inner; ++t) yrow[t] += v * xrow[t];
        }
      }
    } else {
      for (int i = 0; i < m; ++i) {
        const double* xrow = xin + std::int64_t(i) * inner;
        const double* vals = ld.ts_vals + ld.ts_row_off[i];
        for (int k = 0; k < ld.ts_row_len[i]; ++k) {
          const double v = vals[k];
          double* ycol = yout + std::int64_t(ld.ts_row_start[i] + k) * inner;
          for (std::int64_t t = 0; t < inner; ++t) ycol[t] += v * xrow[t];
        }
      }
    }
  }
  return y;
}

// ---------------------------------------------------------------- smoother
// FastDiagonalSolver::solve (tensor.cpp:132-140)
Vec fd_solve(const pmg_piece_desc& pc, const Vec& rhs) {
  std::vector<int> dims(pc.dims, pc.dims + pc.naxes);
  Vec w = rhs;
  for (int a = 0; a < pc.naxes; ++a) w = dense_along(pc.V[a], pc.dims[a], w, dims, a, true);
  for (std::size_t i = 0; i < w.size(); ++i) w[i] /= pc.diag[i];
  for (int a = 0; a < pc.naxes; ++a) w = dense_along(pc.V[a], pc.dims[a], w, dims, a, false);
  return w;
}

// BandedCholesky::solve (banded.cpp:61-77)
Vec banded_solve(const pmg_piece_desc& pc, const Vec& rhs) {
  const int n = pc.chol_dim, bw = pc.chol_bw, w = bw + 1;
  const double* l = pc.chol_l;
  Vec y(static_cast<std::size_t>(n));
  for (int i = 0; i < n; ++i) {
    double s = rhs[i];
    for (int k = std::max(0, i - bw); k < i; ++k) s -= l[std::size_t(i) * w + (i - k)] * y[k];
    y[i] = s / l[std::size_t(i) * w];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = y[i];
    for (int k = i + 1; k < std::min(n, i + bw + 1); ++k) s -= l[std::size_t(k) * w + (k - i)] * y[k];
    y[i] = s / l[std::size_t(i) * w];
  }
  return y;
}

// PieceSmoother::apply_add (smoother.cpp:34-44); `dofs` may be reindexed.
void piece_apply_add(const pmg_piece_desc& pc, const std::int32_t* dofs, const Vec& residual, Vec& corr) {
  if (pc.kind == PMG_PIECE_VERTEX) {
    corr[dofs[0]] += residual[dofs[0]] / pc.scalar;
    return;
  }
  Vec local(static_cast<std::size_t>(pc.ndofs));
  for (std::int64_t i = 0; i < pc.ndofs; ++i) local[i] = residual[dofs[i]];
  if (pc.kind == PMG_PIECE_EDGE && std::int64_t(pc.chol_dim) != pc.ndofs)
    throw DomainError("piece smoother: local vector size mismatch");
  Vec x = pc.kind == PMG_PIECE_EDGE ? banded_solve(pc, local) : fd_solve(pc, local);
  for (std::int64_t i = 0; i < pc.ndofs; ++i) corr[dofs[i]] += x[i];
}

// HybridSmoother::apply (smoother.cpp:110-115)
Vec smoother_apply(const Hier& H, int level, const Vec& r) {
  const Level& L = H.lv[level];
  if (std::int64_t(r.size()) != L.N) throw DomainError("smoother: residual size mismatch");
  Vec corr(std::size_t(L.N), 0.0);
  for (int i = 0; i < L.desc->num_pieces; ++i) {
    const pmg_piece_desc& pc = L.desc->pieces[i];
    piece_apply_add(pc, pc.dofs, r, corr);
  }
  return corr;
}

// ---------------------------------------------------------------- transfer
// TransferOperator::prolong_patch (transfer.cpp:21-38)
Vec prolong_patch(const Hier& H, int level, int k, const Vec& coarse_acc) {
  const Level& Lc = H.lv[level - 1];
  const Level& Lf = H.lv[level];
  Vec work(static_cast<std::size_t>(Lc.S));
  const std::int32_t* l2g = Lc.l2g + k * Lc.S;
  for (std::int64_t f = 0; f < Lc.S; ++f) work[f] = l2g[f] >= 0 ? coarse_acc[l2g[f]] : 0.0;
  std::vector<int> dims(H.d, Lc.ext);
  for (int a = 0; a < H.d; ++a) {
    work = ts_along(Lf, work, dims, a, false);
    dims[a] = Lf.desc->ts_fine_dim;
  }
  return work;
}

// TransferOperator::restrict_patch (transfer.cpp:54-66)
Vec restrict_patch(const Hier& H, int level, const Vec& share) {
  const Level& Lf = H.lv[level];
  std::vector<int> dims(H.d, Lf.ext);
  Vec work = share;
  for (int a = 0; a < H.d; ++a) {
    work = ts_along(Lf, work, dims, a, true);
    dims[a] = Lf.desc->ts_coarse_dim;
  }
  return work;
}

// TransferOperator::prolong, owner-write (transfer.cpp:40-52)
Vec prolong(const Hier& H, int level, const Vec& coarse_acc) {
  const Level& Lf = H.lv[level];
  Vec out(std::size_t(Lf.N), 0.0);
  for (int k = 0; k < H.K; ++k) {
    Vec lat = prolong_patch(H, level, k, coarse_acc);
    const std::int32_t* l2g = Lf.l2g + k * Lf.S;
    for (std::int64_t f = 0; f < Lf.S; ++f) {
      const std::int32_t g = l2g[f];
      if (g >= 0 && Lf.owner_patch(g) == k) out[g] = lat[f];
    }
  }
  return out;
}

// TransferOperator::restrict_full, owner-masked shares (transfer.cpp:68-91)
Vec restrict_full(const Hier& H, int level, const Vec& fine) {
  const Level& Lf = H.lv[level];
  const Level& Lc = H.lv[level - 1];
  Vec out(static_cast<std::size_t>(Lc.N), 0.0), share(std::size_t(Lf.S));
  for (int k = 0; k < H.K; ++k) {
    const std::int32_t* l2gf = Lf.l2g + k * Lf.S;
    for (std::int64_t f = 0; f < Lf.S; ++f) {
      const std::int32_t g = l2gf[f];
      share[f] = (g >= 0 && Lf.owner_patch(g) == k) ? fine[g] : 0.0;
    }
    Vec cs = restrict_patch(H, level, share);
    const std::int32_t* l2gc = Lc.l2g + k * Lc.S;
    for (std::int64_t c = 0; c < Lc.S; ++c)
      if (l2gc[c] >= 0) out[l2gc[c]] += cs[c];
  }
  return out;
}

// Hierarchy::coarse_solve with the dense LLT (multigrid.cpp:52-55)
Vec coarse_solve(const Hier& H, const Vec& rhs) {
  const int n = H.n0;
  const double* L = H.L0;
  if (H.coarse_mode == 1) {
    Vec y(std::size_t(n), 0.0);
    for (int i = 0; i < n; ++i) {
      double s = 0.0;
      for (int k = 0; k < n; ++k) s += H.Ainv[std::size_t(i) * n + k] * rhs[k];
      y[i] = s;
    }
    return y;
  }
  Vec x = rhs;
  for (int i = 0; i < n; ++i) {
    double s = x[i];
    for (int k = 0; k < i; ++k) s -= L[std::size_t(k) * n + i] * x[k];
    x[i] = s / L[std::size_t(i) * n + i];
  }
  for (int i = n - 1; i >= 0; --i) {
    double s = x[i];
    for (int k = i + 1; k < n; ++k) s -= L[std::size_t(i) * n + k] * x[k];
    x[i] = s / L[std::size_t(i) * n + i];
  }
  return x;
}

double vdot(const Vec& a, const Vec& b) {
  double s = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i) s += a[i] * b[i];
  return s;
}

// ---------------------------------------------------------------- serial backend
// SerialBackend (multigrid.hpp:80-114)
struct SerialBackend {
  using AccVec = Vec;
  using DistVec = Vec;
  const Hier* h;
  const pmg_cycle_params& params() const { return h->prm; }
  int finest_level() const { return h->finest(); }
  AccVec zero_acc(int level) const { return Vec(std::size_t(h->lv[level].N), 0.0); }
  DistVec apply_op(int level, const AccVec& u) const { return op_apply(*h, level, u); }
  DistVec residual(int level, const DistVec& f, const AccVec& u) const {
    Vec au = op_apply(*h, level, u);
    Vec r(f.size());
    for (std::size_t i = 0; i < f.size(); ++i) r[i] = f[i] - au[i];
    return r;
  }
  AccVec accumulate(int, const DistVec& r) const { return r; }
  AccVec smooth(int level, const DistVec& r) const { return smoother_apply(*h, level, r); }
  DistVec restrict_residual(int level, const DistVec& r) const { return restrict_full(*h, level, r); }
  void add_prolonged(int level, const AccVec& coarse, double c, AccVec& u) const {
    Vec pu = prolong(*h, level, coarse);
    for (std::size_t i = 0; i < u.size(); ++i) u[i] += c * pu[i];
  }
  AccVec coarse_solve(const DistVec& r) const { return oracle::coarse_solve(*h, r); }
  double dot(int, const DistVec& a, const AccVec& b) const { return vdot(a, b); }
  void axpy_acc(double a, const AccVec& x, AccVec& y) const {
    for (std::size_t i = 0; i < y.size(); ++i) y[i] += a * x[i];
  }
  void axpy_dist(double a, const DistVec& x, DistVec& y) const {
    for (std::size_t i = 0; i < y.size(); ++i) y[i] += a * x[i];
  }
  void xpay_acc(const AccVec& z, double beta, AccVec& p) const {
    for (std::size_t i = 0; i < p.size(); ++i) p[i] = z[i] + beta * p[i];
  }
};

// ---------------------------------------------------------------- templates
// mg_cycle_generic (multigrid.hpp:120-141)
template <class B>
void mg_cycle_generic(const B& b, int level, typename B::AccVec& u, const typename B::DistVec& f) {
  const pmg_cycle_params& prm = b.params();
  for (int i = 0; i < prm.nu; ++i) {
    typename B::AccVec z = b.smooth(level, b.residual(level, f, u));
    b.axpy_acc(prm.tau, z, u);
  }
  typename B::DistVec rc = b.restrict_residual(level, b.residual(level, f, u));
  typename B::AccVec p;
  if (level == 1) {
    p = b.coarse_solve(rc);
  } else {
    p = b.zero_acc(level - 1);
    for (int i = 0; i < prm.mu; ++i) mg_cycle_generic(b, level - 1, p, rc);
  }
  b.add_prolonged(level, p, prm.damp_coarse ? prm.tau : 1.0, u);
  for (int i = 0; i < prm.nu; ++i) {
    typename B::AccVec z = b.smooth(level, b.residual(level, f, u));
    b.axpy_acc(prm.tau, z, u);
  }
}

// mg_precondition (multigrid.hpp:144-149)
template <class B>
typename B::AccVec mg_precondition(const B& b, const typename B::DistVec& r) {
  typename B::AccVec z = b.zero_acc(b.finest_level());
  mg_cycle_generic(b, b.finest_level(), z, r);
  return z;
}

// pcg_generic (multigrid.hpp:155-189); allow_cap turns the divergence throw
// into a normal return for bounded benchmark samples.
template <class B, class P>
typename B::AccVec pcg_generic(const B& b, const typename B::DistVec& f, double tol, int max_iter, const P& precond,
                               std::vector<double>& history, bool allow_cap) {
  const int L = b.finest_level();
  typename B::AccVec u = b.zero_acc(L);
  typename B::DistVec r = f;
  auto norm2 = [&](const typename B::DistVec& v) { return std::sqrt(b.dot(L, v, b.accumulate(L, v))); };
  const double r0 = norm2(r);
  history.clear();
  history.push_back(r0);
  if (r0 == 0.0) return u;
  typename B::AccVec z = precond(r);
  typename B::AccVec p = z;
  double rz = b.dot(L, r, z);
  for (int k = 1; k <= max_iter; ++k) {
    typename B::DistVec Ap = b.apply_op(L, p);
    const double pAp = b.dot(L, Ap, p);
    if (!(pAp > 0.0)) throw DefinitenessError("pcg: search direction with nonpositive energy");
    const double alpha = rz / pAp;
    b.axpy_acc(alpha, p, u);
    b.axpy_dist(-alpha, Ap, r);
    const double rn = norm2(r);
    history.push_back(rn);
    if (rn <= tol * r0) return u;
    if (k == max_iter && allow_cap) return u;
    z = precond(r);
    const double rz_next = b.dot(L, r, z);
    b.xpay_acc(z, rz_next / rz, p);
    rz = rz_next;
  }
  throw DivergenceError("pcg: no convergence within the iteration limit");
}

// ---------------------------------------------------------------- communication
// Communicator / InProcHub / InProcComm (parallel.hpp:31-113, parallel.cpp:21-179)
class Hub {
 public:
  explicit Hub(int ranks) : R(ranks), channels(std::size_t(ranks) * ranks) {}
  const int R;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<std::deque<std::pair<int, Vec>>> channels;
  struct Slot {
    std::vector<Vec> parts;
    int provided = 0, consumed = 0;
  };
  std::map<std::uint64_t, Slot> slots;
  std::uint64_t bytes = 0;
  bool poisoned = false;
  std::string reason;
  bool poison(const std::string& why) {
    std::lock_guard<std::mutex> lock(mu);
    if (poisoned) return false;
    poisoned = true;
    reason = why;
    cv.notify_all();
    return true;
  }
};

class Comm {
 public:
  Comm(Hub* hub, int rank) : hub_(hub), rank_(rank) {}
  int rank() const { return rank_; }
  int size() const { return hub_->R; }
  void send(int dest, int tag, const Vec& data) {
    if (dest < 0 || dest >= size() || dest == rank_) throw TransportError("send: destination is not a peer");
    std::lock_guard<std::mutex> lock(hub_->mu);
    if (hub_->poisoned) throw TransportError(hub_->reason);
    hub_->channels[std::size_t(rank_) * size() + dest].emplace_back(tag, data);
    hub_->bytes += data.size() * 8;
    hub_->cv.notify_all();
  }
  Vec recv(int source, int tag) {
    if (source < 0 || source >= size() || source == rank_) throw TransportError("recv: source is not a peer");
    std::unique_lock<std::mutex> lock(hub_->mu);
    auto& q = hub_->channels[std::size_t(source) * size() + rank_];
    hub_->cv.wait(lock, [&] { return hub_->poisoned || !q.empty(); });
    if (hub_->poisoned) throw TransportError(hub_->reason);
    if (q.front().first != tag) {
      hub_->poisoned = true;
      hub_->reason = "recv: tag mismatch on ordered channel";
      hub_->cv.notify_all();
      throw TransportError(hub_->reason);
    }
    Vec out = std::move(q.front().second);
    q.pop_front();
    return out;
  }
  std::vector<Vec> allgather(const Vec& local) {
    const std::uint64_t seq = next_++;
    std::unique_lock<std::mutex> lock(hub_->mu);
    if (hub_->poisoned) throw TransportError(hub_->reason);
    Hub::Slot& slot = hub_->slots[seq];
    if (slot.parts.empty()) slot.parts.resize(std::size_t(size()));
    slot.parts[rank_] = local;
    slot.provided++;
    hub_->bytes += local.size() * 8 * std::uint64_t(size() - 1);
    hub_->cv.notify_all();
    hub_->cv.wait(lock, [&] { return hub_->poisoned || slot.provided == size(); });
    if (hub_->poisoned) throw TransportError(hub_->reason);
    std::vector<Vec> out = slot.parts;
    if (++slot.consumed == size()) hub_->slots.erase(seq);
    return out;
  }
  // ascending-rank sums (parallel.cpp:21-35)
  double allreduce_sum(double local) {
    std::vector<Vec> parts = allgather(Vec{local});
    double s = parts[0][0];
    for (std::size_t r = 1; r < parts.size(); ++r) s += parts[r][0];
    return s;
  }
  Vec allreduce_sum(const Vec& local) {
    std::vector<Vec> parts = allgather(local);
    Vec s = parts[0];
    for (std::size_t r = 1; r < parts.size(); ++r)
      for (std::size_t i = 0; i < s.size(); ++i) s[i] += parts[r][i];
    return s;
  }

 private:
  Hub* hub_;
  int rank_;
  std::uint64_t next_ = 0;
};

// ---------------------------------------------------------------- parallel backend
struct Partition {  // contiguous_partition (parallel.cpp:181-198)
  int ranks = 1;
  std::vector<int> patch_to_rank;
  std::vector<std::vector<int>> owned;
};

Partition contiguous_partition(int num_patches, int ranks) {
  if (ranks < 1) throw ConfigError("partition: need at least one rank");
  if (ranks > 64) throw ConfigError("partition: rank cap exceeded");
  if (ranks > num_patches) throw ConfigError("partition: more ranks than patches");
  Partition p;
  p.ranks = ranks;
  p.patch_to_rank.resize(num_patches);
  p.owned.resize(ranks);
  for (int r = 0; r < ranks; ++r) {
    const int lo = int(std::int64_t(num_patches) * r / ranks);
    const int hi = int(std::int64_t(num_patches) * (r + 1) / ranks);
    for (int k = lo; k < hi; ++k) {
      p.patch_to_rank[k] = r;
      p.owned[r].push_back(k);
    }
  }
  return p;
}

struct RankLayout {  // parallel.cpp:200-237
  std::vector<std::int32_t> l2g_local, g2l, owner_patch, shared_local;
  std::vector<std::vector<int>> sharers;
  struct Neighbor {
    int rank;
    std::vector<std::int32_t> local;
  };
  std::vector<Neighbor> neighbors;
  RankLayout(const Level& L, int K, const Partition& part, int rank) {
    g2l.assign(std::size_t(L.N), -1);
    std::vector<char> mine(std::size_t(L.N), 0);
    for (int k : part.owned[rank])
      for (std::int64_t f = 0; f < L.S; ++f) {
        const std::int32_t g = L.l2g[k * L.S + f];
        if (g >= 0) mine[g] = 1;
      }
    (void)K;
    for (std::int64_t g = 0; g < L.N; ++g)
      if (mine[g]) {
        g2l[g] = std::int32_t(l2g_local.size());
        l2g_local.push_back(std::int32_t(g));
      }
    owner_patch.resize(l2g_local.size());
    std::vector<std::vector<std::int32_t>> plan(part.ranks);
    for (std::size_t i = 0; i < l2g_local.size(); ++i) {
      const std::int32_t g = l2g_local[i];
      std::int32_t owned_owner = -1;
      std::vector<int> sh;
      for (std::int32_t q = L.rep_off[g]; q < L.rep_off[g + 1]; ++q) {
        const int r = part.patch_to_rank[L.rep_patch[q]];
        if (owned_owner < 0 && r == rank) owned_owner = L.rep_patch[q];
        sh.push_back(r);
      }
      std::sort(sh.begin(), sh.end());
      sh.erase(std::unique(sh.begin(), sh.end()), sh.end());
      owner_patch[i] = owned_owner;
      if (sh.size() > 1) {
        shared_local.push_back(std::int32_t(i));
        sharers.push_back(sh);
        for (int r : sh)
          if (r != rank) plan[r].push_back(std::int32_t(i));
      }
    }
    for (int r = 0; r < part.ranks; ++r)
      if (!plan[r].empty()) neighbors.push_back({r, std::move(plan[r])});
  }
  std::int64_t num_local() const { return std::int64_t(l2g_local.size()); }
};

struct AccV { Vec v; };
struct DistV { Vec v; };

// ParallelBackend (parallel.cpp:247-468)
class ParallelBackend {
 public:
  using AccVec = AccV;
  using DistVec = DistV;
  ParallelBackend(const Hier& h, const Partition& part, Comm& comm) : h_(&h), part_(part), comm_(&comm), rank_(comm.rank()) {
    if (part_.ranks != comm.size()) throw ConfigError("backend: partition and communicator disagree on rank count");
    const int nl = int(h.lv.size());
    layouts_.resize(nl);
    pieces_.resize(nl);
    for (int l = 0; l < nl; ++l) {
      for (int r = 0; r < part_.ranks; ++r) layouts_[l].emplace_back(h.lv[l], h.K, part_, r);
      const RankLayout& lay = layouts_[l][rank_];
      const pmg_level_desc& ld = *h.lv[l].desc;
      for (int i = 0; i < ld.num_pieces; ++i) {
        const pmg_piece_desc& pc = ld.pieces[i];
        std::size_t here = 0;
        for (std::int64_t q = 0; q < pc.ndofs; ++q)
          if (lay.g2l[pc.dofs[q]] >= 0) here++;
        if (here == 0) continue;
        if (here != std::size_t(pc.ndofs)) throw DomainError("backend: a smoother piece straddles the rank boundary");
        std::vector<std::int32_t> local(std::size_t(pc.ndofs));
        for (std::int64_t q = 0; q < pc.ndofs; ++q) local[q] = lay.g2l[pc.dofs[q]];
        pieces_[l].push_back({&pc, std::move(local)});
      }
    }
  }
  const pmg_cycle_params& params() const { return h_->prm; }
  int finest_level() const { return h_->finest(); }
  const RankLayout& layout(int l) const { return layouts_[l][rank_]; }
  AccV zero_acc(int l) const { return AccV{Vec(std::size_t(layout(l).num_local()), 0.0)}; }

  DistV apply_op(int level, const AccV& u) const {
    const RankLayout& lay = layout(level);
    const Level& L = h_->lv[level];
    Vec out(std::size_t(lay.num_local()), 0.0), xl, yl;
    for (int k : part_.owned[rank_]) {
      const std::int32_t* l2g = L.l2g + k * L.S;
      xl.assign(std::size_t(L.S), 0.0);
      yl.assign(std::size_t(L.S), 0.0);
      for (std::int64_t f = 0; f < L.S; ++f)
        if (l2g[f] >= 0) xl[f] = u.v[lay.g2l[l2g[f]]];
      patch_apply_add(*h_, L, k, xl.data(), yl.data());
      for (std::int64_t f = 0; f < L.S; ++f)
        if (l2g[f] >= 0) out[lay.g2l[l2g[f]]] += yl[f];
    }
    return DistV{std::move(out)};
  }
  DistV residual(int level, const DistV& f, const AccV& u) const {
    DistV au = apply_op(level, u);
    Vec r(f.v.size());
    for (std::size_t i = 0; i < r.size(); ++i) r[i] = f.v[i] - au.v[i];
    return DistV{std::move(r)};
  }
  // neighbour exchange, ascending-rank sums (parallel.cpp:306-337)
  AccV accumulate(int level, const DistV& r) const {
    const RankLayout& lay = layout(level);
    const int tag = tag_++;
    Vec out = r.v;
    for (const auto& nb : lay.neighbors) {
      Vec buf(nb.local.size());
      for (std::size_t i = 0; i < nb.local.size(); ++i) buf[i] = r.v[nb.local[i]];
      comm_->send(nb.rank, tag, buf);
    }
    std::vector<Vec> in(lay.neighbors.size());
    std::vector<int> index_of(part_.ranks, -1);
    for (std::size_t j = 0; j < lay.neighbors.size(); ++j) {
      in[j] = comm_->recv(lay.neighbors[j].rank, tag);
      index_of[lay.neighbors[j].rank] = int(j);
    }
    std::vector<std::size_t> cursor(lay.neighbors.size(), 0);
    for (std::size_t s = 0; s < lay.shared_local.size(); ++s) {
      const std::int32_t li = lay.shared_local[s];
      double sum = 0.0;
      for (int rr : lay.sharers[s]) {
        if (rr == rank_)
          sum += r.v[li];
        else {
          const int j = index_of[rr];
          sum += in[j][cursor[j]++];
        }
      }
      out[li] = sum;
    }
    return AccV{std::move(out)};
  }
  Vec apply_pieces_values(int level, const Vec& v) const {
    Vec z(std::size_t(layout(level).num_local()), 0.0);
    for (const auto& [pc, local] : pieces_[level]) piece_apply_add(*pc, local.data(), v, z);
    return z;
  }
  AccV smooth(int level, const DistV& r) const { return accumulate(level, DistV{apply_pieces_values(level, r.v)}); }
  // parallel.cpp:357-382
  DistV restrict_residual(int level, const DistV& r) const {
    const RankLayout& lf = layout(level);
    const RankLayout& lc = layout(level - 1);
    const Level& Lf = h_->lv[level];
    const Level& Lc = h_->lv[level - 1];
    Vec out(static_cast<std::size_t>(lc.num_local()), 0.0), share(std::size_t(Lf.S));
    for (int k : part_.owned[rank_]) {
      const std::int32_t* l2gf = Lf.l2g + k * Lf.S;
      std::fill(share.begin(), share.end(), 0.0);
      for (std::int64_t f = 0; f < Lf.S; ++f) {
        const std::int32_t g = l2gf[f];
        if (g < 0) continue;
        const std::int32_t li = lf.g2l[g];
        if (lf.owner_patch[li] == k) share[f] = r.v[li];
      }
      Vec cs = restrict_patch(*h_, level, share);
      const std::int32_t* l2gc = Lc.l2g + k * Lc.S;
      for (std::int64_t c = 0; c < Lc.S; ++c)
        if (l2gc[c] >= 0) out[lc.g2l[l2gc[c]]] += cs[c];
    }
    return DistV{std::move(out)};
  }
  // parallel.cpp:384-409
  void add_prolonged(int level, const AccV& coarse, double c, AccV& u) const {
    const RankLayout& lf = layout(level);
    const RankLayout& lc = layout(level - 1);
    const Level& Lf = h_->lv[level];
    Vec scratch(std::size_t(h_->lv[level - 1].N), 0.0);
    for (std::int64_t i = 0; i < lc.num_local(); ++i) scratch[lc.l2g_local[i]] = coarse.v[i];
    Vec pu(std::size_t(lf.num_local()), 0.0);
    for (int k : part_.owned[rank_]) {
      Vec lat = prolong_patch(*h_, level, k, scratch);
      const std::int32_t* l2g = Lf.l2g + k * Lf.S;
      for (std::int64_t f = 0; f < Lf.S; ++f) {
        const std::int32_t g = l2g[f];
        if (g < 0) continue;
        const std::int32_t li = lf.g2l[g];
        if (lf.owner_patch[li] == k) pu[li] = lat[f];
      }
    }
    for (std::size_t i = 0; i < u.v.size(); ++i) u.v[i] += c * pu[i];
  }
  // parallel.cpp:411-422
  AccV coarse_solve(const DistV& r) const {
    const RankLayout& lay = layout(0);
    Vec scattered(std::size_t(h_->lv[0].N), 0.0);
    for (std::int64_t i = 0; i < lay.num_local(); ++i) scattered[lay.l2g_local[i]] = r.v[i];
    Vec global = comm_->allreduce_sum(scattered);
    Vec sol = oracle::coarse_solve(*h_, global);
    Vec out(static_cast<std::size_t>(lay.num_local()));
    for (std::int64_t i = 0; i < lay.num_local(); ++i) out[i] = sol[lay.l2g_local[i]];
    return AccV{std::move(out)};
  }
  double dot(int, const DistV& a, const AccV& b) const { return comm_->allreduce_sum(vdot(a.v, b.v)); }
  void axpy_acc(double a, const AccV& x, AccV& y) const {
    for (std::size_t i = 0; i < y.v.size(); ++i) y.v[i] += a * x.v[i];
  }
  void axpy_dist(double a, const DistV& x, DistV& y) const {
    for (std::size_t i = 0; i < y.v.size(); ++i) y.v[i] += a * x.v[i];
  }
  void xpay_acc(const AccV& z, double beta, AccV& p) const {
    for (std::size_t i = 0; i < p.v.size(); ++i) p.v[i] = z.v[i] + beta * p.v[i];
  }
  DistV to_distributed_owner(int level, const Vec& global) const {  // parallel.cpp:436-446
    const RankLayout& lay = layout(level);
    const Level& L = h_->lv[level];
    Vec out(std::size_t(lay.num_local()), 0.0);
    for (std::int64_t i = 0; i < lay.num_local(); ++i) {
      const std::int32_t g = lay.l2g_local[i];
      if (part_.patch_to_rank[L.owner_patch(g)] == rank_) out[i] = global[g];
    }
    return DistV{std::move(out)};
  }
  Vec gather_global(int level, const AccV& u) const {  // parallel.cpp:448-457
    std::vector<Vec> parts = comm_->allgather(u.v);
    Vec out(std::size_t(h_->lv[level].N), 0.0);
    for (int r = 0; r < part_.ranks; ++r) {
      const RankLayout& lay = layouts_[level][r];
      for (std::int64_t i = 0; i < lay.num_local(); ++i) out[lay.l2g_local[i]] = parts[r][i];
    }
    return out;
  }

 private:
  const Hier* h_;
  Partition part_;
  Comm* comm_;
  int rank_;
  std::vector<std::vector<RankLayout>> layouts_;
  std::vector<std::vector<std::pair<const pmg_piece_desc*, std::vector<std::int32_t>>>> pieces_;
  mutable int tag_ = 0;
};

}  // namespace oracle

// ================================================================ C ABI
using namespace oracle;

struct oracle_ctx {
  Hier h;
};

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PMG_OK;
  } catch (const ConfigError& e) {
    g_err = e.what();
    return PMG_ERR_CONFIG;
  } catch (const DivergenceError& e) {
    g_err = e.what();
    return PMG_ERR_DIVERGENCE;
  } catch (const TransportError& e) {
    g_err = e.what();
    return PMG_ERR_TRANSPORT;
  } catch (const DomainError& e) {
    g_err = e.what();
    return PMG_ERR_DOMAIN;
  } catch (const DefinitenessError& e) {
    g_err = e.what();
    return PMG_ERR_DEFINITENESS;
  } catch (const std::exception& e) {
    g_err = e.what();
    return PMG_ERR_GENERIC;
  }
}

Vec to_vec(const double* p, std::int64_t n) { return Vec(p, p + n); }
void from_vec(const Vec& v, double* out) { std::memcpy(out, v.data(), v.size() * sizeof(double)); }

void check_level(const Hier& h, int level, int lo) {
  if (level < lo || level > h.finest()) throw DomainError("oracle: level out of range");
}
}  // namespace

extern "C" {

const char* oracle_last_error(void) { return g_err.c_str(); }

int oracle_create(const pmg_hierarchy_desc* desc, oracle_ctx** out) {
  return guarded([&] {
    auto c = std::make_unique<oracle_ctx>();
    build_view(desc, c->h);
    *out = c.release();
  });
}

void oracle_destroy(oracle_ctx* ctx) { delete ctx; }

int64_t oracle_num_dofs(oracle_ctx* ctx, int level) { return ctx->h.lv[level].N; }

int oracle_apply_op(oracle_ctx* ctx, int level, const double* u, double* out) {
  return guarded([&] {
    check_level(ctx->h, level, 0);
    from_vec(op_apply(ctx->h, level, to_vec(u, ctx->h.lv[level].N)), out);
  });
}

int oracle_residual(oracle_ctx* ctx, int level, const double* f, const double* u, double* out) {
  return guarded([&] {
    check_level(ctx->h, level, 0);
    SerialBackend b{&ctx->h};
    const std::int64_t n = ctx->h.lv[level].N;
    from_vec(b.residual(level, to_vec(f, n), to_vec(u, n)), out);
  });
}

int oracle_smooth(oracle_ctx* ctx, int level, const double* r, double* out) {
  return guarded([&] {
    check_level(ctx->h, level, 0);
    from_vec(smoother_apply(ctx->h, level, to_vec(r, ctx->h.lv[level].N)), out);
  });
}

int oracle_restrict(oracle_ctx* ctx, int level, const double* r, double* out_coarse) {
  return guarded([&] {
    check_level(ctx->h, level, 1);
    from_vec(restrict_full(ctx->h, level, to_vec(r, ctx->h.lv[level].N)), out_coarse);
  });
}

int oracle_add_prolonged(oracle_ctx* ctx, int level, const double* coarse, double c, double* u) {
  return guarded([&] {
    check_level(ctx->h, level, 1);
    SerialBackend b{&ctx->h};
    Vec uu = to_vec(u, ctx->h.lv[level].N);
    b.add_prolonged(level, to_vec(coarse, ctx->h.lv[level - 1].N), c, uu);
    from_vec(uu, u);
  });
}

int oracle_set_coarse_mode(oracle_ctx* ctx, int mode) {
  return guarded([&] {
    if (mode != 0 && mode != 1) throw ConfigError("coarse mode must be 0 (LLT) or 1 (explicit inverse)");
    Hier& H = ctx->h;
    if (mode == 1 && H.Ainv.empty()) {
      // A0^-1 = L^-T L^-1 from the column-major lower factor
      const int n = H.n0;
      const double* L = H.L0;
      std::vector<double> Li(std::size_t(n) * n, 0.0);  // column-major lower inverse
      for (int j = 0; j < n; ++j) {
        Li[std::size_t(j) * n + j] = 1.0 / L[std::size_t(j) * n + j];
        for (int i = j + 1; i < n; ++i) {
          double s = 0.0;
          for (int k = j; k < i; ++k) s += L[std::size_t(k) * n + i] * Li[std::size_t(j) * n + k];
          Li[std::size_t(j) * n + i] = -s / L[std::size_t(i) * n + i];
        }
      }
      H.Ainv.assign(std::size_t(n) * n, 0.0);
      for (int i = 0; i < n; ++i)
        for (int j = 0; j <= i; ++j) {
          double s = 0.0;
          for (int k = i; k < n; ++k) s += Li[std::size_t(i) * n + k] * Li[std::size_t(j) * n + k];
          H.Ainv[std::size_t(i) * n + j] = H.Ainv[std::size_t(j) * n + i] = s;
        }
    }
    H.coarse_mode = mode;
  });
}

int oracle_coarse_solve(oracle_ctx* ctx, const double* r, double* out) {
  return guarded([&] { from_vec(coarse_solve(ctx->h, to_vec(r, ctx->h.n0)), out); });
}

int oracle_mg_cycle(oracle_ctx* ctx, int level, double* u, const double* f) {
  return guarded([&] {
    check_level(ctx->h, level, 1);
    SerialBackend b{&ctx->h};
    const std::int64_t n = ctx->h.lv[level].N;
    Vec uu = to_vec(u, n);
    mg_cycle_generic(b, level, uu, to_vec(f, n));
    from_vec(uu, u);
  });
}

int oracle_precondition(oracle_ctx* ctx, const double* r, double* z) {
  return guarded([&] {
    SerialBackend b{&ctx->h};
    from_vec(mg_precondition(b, to_vec(r, ctx->h.lv[ctx->h.finest()].N)), z);
  });
}

int oracle_pcg_solve(oracle_ctx* ctx, const double* f, double tol, int max_iter, int allow_cap, double* u,
                     double* history, int* iterations, double* t_solve) {
  return guarded([&] {
    SerialBackend b{&ctx->h};
    std::vector<double> hist;
    const Vec ff = to_vec(f, ctx->h.lv[ctx->h.finest()].N);
    auto t0 = std::chrono::steady_clock::now();
    Vec uu = pcg_generic(b, ff, tol, max_iter, [&](const Vec& r) { return mg_precondition(b, r); }, hist,
                         allow_cap != 0);
    const double ts = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    from_vec(uu, u);
    std::copy(hist.begin(), hist.end(), history);
    *iterations = int(hist.size()) - 1;
    if (t_solve) *t_solve = ts;
  });
}

int oracle_parallel_pcg_solve(oracle_ctx* ctx, int ranks, const double* f, double tol, int max_iter, int allow_cap,
                              double* u, double* history, int* iterations, double* t_solve, uint64_t* comm_bytes) {
  return guarded([&] {
    const Hier& h = ctx->h;
    const Partition part = contiguous_partition(h.K, ranks);
    Hub hub(ranks);
    const int L = h.finest();
    const Vec fg = to_vec(f, h.lv[L].N);
    Vec ug;
    std::vector<double> hist0;
    double ts0 = 0.0;
    std::vector<std::exception_ptr> errors(ranks);
    std::atomic<int> primary{-1};
    std::vector<std::thread> threads;
    // run_ranks (parallel.cpp:153-179) over parallel_solve_rank (parallel.cpp:470-495)
    for (int r = 0; r < ranks; ++r)
      threads.emplace_back([&, r] {
        try {
          Comm comm(&hub, r);
          ParallelBackend b(h, part, comm);
          DistV fd = b.to_distributed_owner(L, fg);
          std::vector<double> hist;
          auto t0 = std::chrono::steady_clock::now();
          AccV uu = pcg_generic(b, fd, tol, max_iter, [&](const DistV& res) { return mg_precondition(b, res); }, hist,
                                allow_cap != 0);
          const double ts = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
          Vec gathered = b.gather_global(L, uu);
          if (r == 0) {
            ug = std::move(gathered);
            hist0 = hist;
            ts0 = ts;
          }
        } catch (...) {
          errors[r] = std::current_exception();
          if (hub.poison("peer rank failed")) {
            int expected = -1;
            primary.compare_exchange_strong(expected, r);
          }
        }
      });
    for (auto& t : threads) t.join();
    const int first = primary.load();
    if (first >= 0 && errors[first]) std::rethrow_exception(errors[first]);
    for (auto& e : errors)
      if (e) std::rethrow_exception(e);
    from_vec(ug, u);
    std::copy(hist0.begin(), hist0.end(), history);
    *iterations = int(hist0.size()) - 1;
    if (t_solve) *t_solve = ts0;
    if (comm_bytes) *comm_bytes = hub.bytes;
  });
}

}  // extern "C"
