// Hierarchy setup: assembly, smoother payloads, transfers, coarse factor,
// load vector and domain generators (see hierarchy.hpp for the reference map).
#include "hierarchy.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <map>
#include <mutex>
#include <sstream>
#include <thread>
#include <tuple>

namespace pmg {

namespace {

double seconds_since(std::chrono::steady_clock::time_point t0) {
  return std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
}

// Deterministic work distribution: items [0, n) handed out in order to
// `threads` workers; each item must be independent of the others.
template <class F>
void parallel_for(std::int64_t n, int threads, F&& f) {
  if (threads <= 1 || n <= 1) {
    for (std::int64_t i = 0; i < n; ++i) f(i);
    return;
  }
  std::atomic<std::int64_t> next{0};
  std::exception_ptr err;
  std::mutex err_mu;
  std::vector<std::thread> pool;
  const int nt = int(std::min<std::int64_t>(threads, n));
  for (int t = 0; t < nt; ++t)
    pool.emplace_back([&] {
      for (;;) {
        const std::int64_t i = next++;
        if (i >= n) break;
        try {
          f(i);
        } catch (...) {
          std::lock_guard<std::mutex> lock(err_mu);
          if (!err) err = std::current_exception();
        }
      }
    });
  for (auto& th : pool) th.join();
  if (err) std::rethrow_exception(err);
}

// Per-direction basis tables at the Gauss points of every element of the
// full space: vals[e][k*q1+q] (assembly.cpp:38-59).
struct BasisTables {
  int q1 = 0, p = 0;
  std::vector<std::vector<double>> vals, ders;
};

BasisTables tabulate(int degree, int elements, const QuadratureRule& rule) {
  BasisTables t;
  t.p = degree;
  t.q1 = int(rule.nodes.size());
  UnivariateSpace space(degree, elements);
  for (int e = 0; e < elements; ++e) {
    std::vector<double> v((degree + 1) * t.q1), d((degree + 1) * t.q1);
    for (int q = 0; q < t.q1; ++q) {
      const double x = (e + rule.nodes[q]) / elements;
      BasisEval bv = eval_basis(space, x, 0);
      BasisEval bd = eval_basis(space, x, 1);
      for (int k = 0; k <= degree; ++k) {
        v[k * t.q1 + q] = bv.values[k];
        d[k * t.q1 + q] = bd.values[k];
      }
    }
    t.vals.push_back(std::move(v));
    t.ders.push_back(std::move(d));
  }
  return t;
}

double det_and_inverse(int d, const double* J, double* Ji) {
  if (d == 2) {
    const double det = J[0] * J[3] - J[1] * J[2];
    Ji[0] = J[3] / det;
    Ji[1] = -J[1] / det;
    Ji[2] = -J[2] / det;
    Ji[3] = J[0] / det;
    return det;
  }
  const double c00 = J[4] * J[8] - J[5] * J[7];
  const double c01 = J[5] * J[6] - J[3] * J[8];
  const double c02 = J[3] * J[7] - J[4] * J[6];
  const double det = J[0] * c00 + J[1] * c01 + J[2] * c02;
  Ji[0] = c00 / det;
  Ji[3] = c01 / det;
  Ji[6] = c02 / det;
  Ji[1] = (J[2] * J[7] - J[1] * J[8]) / det;
  Ji[4] = (J[0] * J[8] - J[2] * J[6]) / det;
  Ji[7] = (J[1] * J[6] - J[0] * J[7]) / det;
  Ji[2] = (J[1] * J[5] - J[2] * J[4]) / det;
  Ji[5] = (J[2] * J[3] - J[0] * J[5]) / det;
  Ji[8] = (J[0] * J[4] - J[1] * J[3]) / det;
  return det;
}

std::uint64_t splitmix64(std::uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

double unit_draw(std::uint64_t seed, std::uint64_t index) {
  const std::uint64_t z = splitmix64(seed ^ (index * 0xD1B54A32D192ED03ull + 0x632BE59BD9B4E019ull));
  return double(z >> 11) * (1.0 / 9007199254740992.0);
}

}  // namespace

double node_uniform(std::uint64_t seed, std::uint64_t index) { return 2.0 * unit_draw(seed, index) - 1.0; }

std::int64_t stored_stiffness_entries(int degree, int elements, int dim, int patches) {
  const int extent = elements + degree;
  std::int64_t pairs = 0;
  for (int i = 0; i < extent; ++i) pairs += std::min(i + degree, extent - 1) - std::max(i - degree, 0) + 1;
  std::int64_t per_patch = 1;
  for (int a = 0; a < dim; ++a) per_patch *= pairs;
  return per_patch * patches;
}

// ============================================================ assembly
void assemble_patch_band(const GeometryMap& geo, int degree, int elements, double* band, int threads) {
  const int d = geo.dim();
  const int p = degree;
  const int ext = elements + degree;
  const QuadratureRule& rule = gauss_legendre(p + 1);
  const int q1 = int(rule.nodes.size());
  const BasisTables tab = tabulate(p, elements, rule);
  int nloc = 1, nq = 1, O = 1;
  std::int64_t S = 1;
  for (int a = 0; a < d; ++a) {
    nloc *= p + 1;
    nq *= q1;
    O *= 2 * p + 1;
    S *= ext;
  }
  std::fill(band, band + std::size_t(O) * std::size_t(S), 0.0);
  std::int64_t layer = 1;  // elements per layer of the slowest axis
  for (int a = 0; a < d - 1; ++a) layer *= elements;
  const int chunk = std::max(p + 1, 4);
  const int nchunks = (elements + chunk - 1) / chunk;
  std::atomic<int> det_sign_seen{0};  // +1 / -1 once fixed

  auto run_chunk = [&](int c) {
    std::vector<double> G(std::size_t(nloc) * d * nq), H(std::size_t(nloc) * d * nq), E(std::size_t(nloc) * nloc);
    std::vector<double> coeff(std::size_t(nq) * d * d);
    double param[3], J[9], Ji[9];
    int ecell[3], qidx[3], li[3], lj[3];
    const int e_lo = c * chunk, e_hi = std::min(elements, (c + 1) * chunk);
    for (std::int64_t e = std::int64_t(e_lo) * layer; e < std::int64_t(e_hi) * layer; ++e) {
      std::int64_t rem = e;
      for (int a = 0; a < d; ++a) {
        ecell[a] = int(rem % elements);
        rem /= elements;
      }
      // quadrature geometry pass (assembly.cpp:161-182)
      for (int a = 0; a < d; ++a) qidx[a] = 0;
      for (int q = 0; q < nq; ++q) {
        double w = 1.0;
        for (int a = 0; a < d; ++a) {
          param[a] = (ecell[a] + rule.nodes[qidx[a]]) / elements;
          w *= rule.weights[qidx[a]] / elements;
        }
        geo.jacobian(param, J);
        const double det = det_and_inverse(d, J, Ji);
        int sgn = det_sign_seen.load();
        if (sgn == 0) {
          int want = det > 0.0 ? 1 : -1;
          det_sign_seen.compare_exchange_strong(sgn, want);
          sgn = det_sign_seen.load();
        }
        if (!(det * sgn > 1e-14)) throw SingularGeometryError("assembly: degenerate or folded geometry map");
        const double s = w * std::abs(det);
        for (int a = 0; a < d; ++a)
          for (int b = 0; b < d; ++b) {
            double m = 0.0;
            for (int k = 0; k < d; ++k) m += Ji[a * d + k] * Ji[b * d + k];
            coeff[(std::size_t(q) * d + a) * d + b] = s * m;
          }
        for (int a = 0; a < d; ++a) {
          if (++qidx[a] < q1) break;
          qidx[a] = 0;
        }
      }
      // gradient tables G(i, a*nq+q) stored at [(a*nq+q)*nloc + i] (assembly.cpp:184-207)
      for (int a = 0; a < d; ++a) li[a] = 0;
      for (int i = 0; i < nloc; ++i) {
        for (int a = 0; a < d; ++a) qidx[a] = 0;
        for (int q = 0; q < nq; ++q) {
          for (int a = 0; a < d; ++a) {
            double g = 1.0;
            for (int b = 0; b < d; ++b) {
              const std::vector<double>& t = (b == a) ? tab.ders[ecell[b]] : tab.vals[ecell[b]];
              g *= t[li[b] * q1 + qidx[b]];
            }
            G[(std::size_t(a) * nq + q) * nloc + i] = g;
          }
          for (int a = 0; a < d; ++a) {
            if (++qidx[a] < q1) break;
            qidx[a] = 0;
          }
        }
        for (int a = 0; a < d; ++a) {
          if (++li[a] <= p) break;
          li[a] = 0;
        }
      }
      // H_a(:, q) = sum_b C_ab(q) G_b(:, q)  (assembly.cpp:209-216)
      for (int a = 0; a < d; ++a)
        for (int q = 0; q < nq; ++q) {
          double* h = &H[(std::size_t(a) * nq + q) * nloc];
          const double* c0 = &coeff[(std::size_t(q) * d + a) * d];
          const double* g0 = &G[std::size_t(q) * nloc];
          for (int i = 0; i < nloc; ++i) h[i] = c0[0] * g0[i];
          for (int b = 1; b < d; ++b) {
            const double* gb = &G[(std::size_t(b) * nq + q) * nloc];
            for (int i = 0; i < nloc; ++i) h[i] += c0[b] * gb[i];
          }
        }
      // E = G H^T stored E[j*nloc + i] (assembly.cpp:218); every entry sums
      // over the d*nq columns in ascending order, register-blocked 4 x 8
      const int ncol = d * nq;
      for (int jb = 0; jb < nloc; jb += 4) {
        const int jn = std::min(4, nloc - jb);
        for (int ib = 0; ib < nloc; ib += 8) {
          const int in = std::min(8, nloc - ib);
          double acc[4][8] = {};
          if (jn == 4 && in == 8) {
            for (int col = 0; col < ncol; ++col) {
              const double* g = &G[std::size_t(col) * nloc + ib];
              const double* h = &H[std::size_t(col) * nloc + jb];
              for (int jj = 0; jj < 4; ++jj)
                for (int ii = 0; ii < 8; ++ii) acc[jj][ii] += g[ii] * h[jj];
            }
          } else {
            for (int col = 0; col < ncol; ++col) {
              const double* g = &G[std::size_t(col) * nloc + ib];
              const double* h = &H[std::size_t(col) * nloc + jb];
              for (int jj = 0; jj < jn; ++jj)
                for (int ii = 0; ii < in; ++ii) acc[jj][ii] += g[ii] * h[jj];
            }
          }
          for (int jj = 0; jj < jn; ++jj)
            for (int ii = 0; ii < in; ++ii) E[std::size_t(jb + jj) * nloc + ib + ii] = acc[jj][ii];
        }
      }
      // scatter into the band (assembly.cpp:220-240)
      for (int a = 0; a < d; ++a) li[a] = 0;
      for (int i = 0; i < nloc; ++i) {
        std::int64_t r = 0;
        for (int a = d - 1; a >= 0; --a) r = r * ext + (ecell[a] + li[a]);
        for (int a = 0; a < d; ++a) lj[a] = 0;
        for (int j = 0; j < nloc; ++j) {
          int o = 0;
          for (int a = d - 1; a >= 0; --a) o = o * (2 * p + 1) + (lj[a] - li[a] + p);
          band[std::size_t(o) * S + r] += E[std::size_t(j) * nloc + i];
          for (int a = 0; a < d; ++a) {
            if (++lj[a] <= p) break;
            lj[a] = 0;
          }
        }
        for (int a = 0; a < d; ++a) {
          if (++li[a] <= p) break;
          li[a] = 0;
        }
      }
    }
  };
  // two colour phases over chunks of element layers: chunks of one colour
  // never touch a common lattice row
  for (int phase = 0; phase < 2; ++phase) {
    const int count = (nchunks - phase + 1) / 2;
    parallel_for(count, threads, [&](std::int64_t i) { run_chunk(int(2 * i + phase)); });
  }
}

std::vector<double> assemble_rhs(const DofMapper& mapper, const RhsSpec& spec, int threads) {
  const MultiPatchDomain& dom = mapper.domain();
  const int d = dom.dim;
  const int p = mapper.degree();
  const int n = mapper.elements();
  const int ext = mapper.extent();
  const QuadratureRule& rule = gauss_legendre(p + 1);
  const int q1 = int(rule.nodes.size());
  const BasisTables tab = tabulate(p, n, rule);
  const int K = dom.num_patches();
  if (spec.zero) return std::vector<double>(std::size_t(mapper.num_dofs()), 0.0);
  std::int64_t ecount = 1, nq = 1;
  for (int a = 0; a < d; ++a) {
    ecount *= n;
    nq *= q1;
  }
  std::vector<std::vector<double>> local(K);
  parallel_for(K, threads, [&](std::int64_t kk) {
    const int k = int(kk);
    const GeometryMap& geo = dom.patches[k];
    std::vector<double>& acc = local[k];
    acc.assign(std::size_t(mapper.lattice_size()), 0.0);
    double det_sign = 0.0;
    double param[3], J[9], Ji[9], x[3];
    int ecell[3] = {0, 0, 0}, qidx[3], li[3];
    for (std::int64_t e = 0; e < ecount; ++e) {
      for (int a = 0; a < d; ++a) qidx[a] = 0;
      for (std::int64_t q = 0; q < nq; ++q) {
        double w = 1.0;
        for (int a = 0; a < d; ++a) {
          param[a] = (ecell[a] + rule.nodes[qidx[a]]) / n;
          w *= rule.weights[qidx[a]] / n;
        }
        geo.jacobian(param, J);
        const double det = det_and_inverse(d, J, Ji);
        if (det_sign == 0.0) det_sign = det > 0.0 ? 1.0 : -1.0;
        if (!(det * det_sign > 1e-14)) throw SingularGeometryError("assembly: degenerate or folded geometry map");
        double fval;
        if (spec.kind == RhsSpec::function) {
          geo.eval(param, x);
          fval = spec.f(x);
        } else {
          fval = node_uniform(spec.seed, (std::uint64_t(k) * std::uint64_t(ecount) + std::uint64_t(e)) *
                                             std::uint64_t(nq) + std::uint64_t(q));
        }
        const double fw = w * std::abs(det) * fval;
        for (int a = 0; a < d; ++a) li[a] = 0;
        for (;;) {
          double v = 1.0;
          std::int64_t flat = 0;
          for (int a = d - 1; a >= 0; --a) {
            v *= tab.vals[ecell[a]][li[a] * q1 + qidx[a]];
            flat = flat * ext + (ecell[a] + li[a]);
          }
          acc[std::size_t(flat)] += fw * v;
          int a = 0;
          for (; a < d; ++a) {
            if (++li[a] <= p) break;
            li[a] = 0;
          }
          if (a == d) break;
        }
        for (int a = 0; a < d; ++a) {
          if (++qidx[a] < q1) break;
          qidx[a] = 0;
        }
      }
      for (int a = 0; a < d; ++a) {
        if (++ecell[a] < n) break;
        ecell[a] = 0;
      }
    }
  });
  std::vector<double> rhs(std::size_t(mapper.num_dofs()), 0.0);
  for (int k = 0; k < K; ++k) {
    const auto& l2g = mapper.local_to_global(k);
    for (std::int64_t f = 0; f < mapper.lattice_size(); ++f)
      if (l2g[f] >= 0) rhs[l2g[f]] += local[k][f];
  }
  return rhs;
}

// ============================================================ hierarchy
namespace {

struct SpaceKey {
  int p, n, l, r;
  bool operator<(const SpaceKey& o) const { return std::tie(p, n, l, r) < std::tie(o.p, o.n, o.l, o.r); }
};

struct EigCache {
  std::mutex mu;
  std::map<SpaceKey, std::pair<std::shared_ptr<const Dense>, std::vector<double>>> map;
  std::pair<std::shared_ptr<const Dense>, std::vector<double>> get(const UnivariateSpace& s) {
    SpaceKey key{s.degree(), s.elements(), int(s.left()), int(s.right())};
    {
      std::lock_guard<std::mutex> lock(mu);
      auto it = map.find(key);
      if (it != map.end()) return it->second;
    }
    Dense K = univariate_stiffness(s).to_dense();
    Dense M = univariate_mass(s).to_dense();
    GenEigDecomposition ge = gen_eig(K, M);
    auto val = std::make_pair(std::make_shared<const Dense>(std::move(ge.eigenvectors)), std::move(ge.eigenvalues));
    std::lock_guard<std::mutex> lock(mu);
    return map.emplace(key, std::move(val)).first->second;
  }
};

// FastDiagonalSolver ctor (tensor.cpp:104-130)
FDPayload make_fd(const std::vector<UnivariateSpace>& spaces, double sigma, double scale, EigCache& cache) {
  FDPayload fd;
  fd.naxes = int(spaces.size());
  std::vector<std::vector<double>> lambdas;
  std::int64_t total = 1;
  for (int a = 0; a < fd.naxes; ++a) {
    auto [V, lam] = cache.get(spaces[a]);
    fd.V[a] = V;
    fd.dims[a] = int(lam.size());
    lambdas.push_back(lam);
    total *= fd.dims[a];
  }
  fd.diag.resize(std::size_t(total));
  int idx[3] = {0, 0, 0};
  for (std::int64_t f = 0; f < total; ++f) {
    double s = sigma;
    for (int a = 0; a < fd.naxes; ++a) s += lambdas[a][idx[a]];
    fd.diag[std::size_t(f)] = scale * s;
    for (int a = 0; a < fd.naxes; ++a) {
      if (++idx[a] < fd.dims[a]) break;
      idx[a] = 0;
    }
  }
  return fd;
}

}  // namespace

Hierarchy::Hierarchy(const MultiPatchDomain& domain, int degree, int n0, int levels, CycleParams params,
                     const RhsSpec& rhs, int threads, bool host_assembly)
    : domain_(std::make_unique<MultiPatchDomain>(domain)), degree_(degree), n0_(n0), params_(params) {
  if (levels < 1) throw ConfigError("hierarchy: need at least one refinement level");
  if (n0 < 1) throw ConfigError("hierarchy: coarsest element count must be positive");
  if (params.nu < 1) throw ConfigError("hierarchy: need at least one smoothing step");
  if (params.mu < 1 || params.mu > 2) throw ConfigError("hierarchy: cycle index must be 1 or 2");
  if (params.tau <= 0.0 || params.sigma_scale <= 0.0)
    throw ConfigError("hierarchy: damping and shift scale must be positive");
  if (degree < 1 || degree > kMaxDegree) throw ConfigError("hierarchy: degree out of range");
  threads = std::max(1, threads);
  const int d = domain_->dim;
  const int K = domain_->num_patches();

  auto t0 = std::chrono::steady_clock::now();
  const bool timing = std::getenv("PMG_SETUP_TIMING") != nullptr;
  double t_map = 0, t_cls = 0, t_pay = 0;
  levels_.resize(levels + 1);
  EigCache cache;
  for (int l = 0; l <= levels; ++l) {
    Level& L = levels_[l];
    L.elements = n0 << l;
    auto ta = std::chrono::steady_clock::now();
    L.mapper = std::make_unique<DofMapper>(*domain_, degree, L.elements);
    t_map += seconds_since(ta);
    const std::int64_t S = L.mapper->lattice_size();
    L.l2g.resize(std::size_t(S) * K);
    for (int k = 0; k < K; ++k)
      std::copy(L.mapper->local_to_global(k).begin(), L.mapper->local_to_global(k).end(), L.l2g.begin() + k * S);
    if (l >= 1) L.two_scale = two_scale_matrix(UnivariateSpace(degree, levels_[l - 1].elements));
    // smoother pieces and payloads (smoother.cpp:84-108)
    const double h = 1.0 / L.elements;
    const double sigma = 1.0 / (params.sigma_scale * h * h);
    auto tb = std::chrono::steady_clock::now();
    std::vector<Piece> pieces = classify_dofs(*L.mapper);
    t_cls += seconds_since(tb);
    auto tc = std::chrono::steady_clock::now();
    L.pieces.resize(pieces.size());
    parallel_for(std::int64_t(pieces.size()), threads, [&](std::int64_t i) {
      Piece& pc = pieces[i];
      PieceData& pd = L.pieces[i];
      pd.kind = pc.kind;
      pd.patch = pc.patch;
      pd.dofs = pc.dofs;
      switch (pc.kind) {
        case PieceKind::interior:
          pd.fd = make_fd(pc.spaces, sigma, 1.0, cache);
          break;
        case PieceKind::face:
          pd.fd = make_fd(pc.spaces, double(degree) * degree / (h * h), h / degree, cache);
          break;
        case PieceKind::edge: {
          const UnivariateSpace& sp = pc.spaces.at(0);
          BandedSymMatrix Kb = univariate_stiffness(sp), Mb = univariate_mass(sp);
          BandedSymMatrix Lb = BandedSymMatrix::combine(std::pow(h / degree, d - 1), Kb, std::pow(h / degree, d - 3), Mb);
          pd.chol = BandedCholesky(Lb);
          break;
        }
        case PieceKind::vertex:
          pd.scalar = std::pow(h / degree, d - 2);
          break;
      }
    });
    t_pay += seconds_since(tc);
  }
  t_setup_ = seconds_since(t0);
  if (timing)
    std::fprintf(stderr, "[pmg setup] DofMapper %.2f s, classify_dofs %.2f s, piece payloads %.2f s (of %.2f s)\n", t_map,
                 t_cls, t_pay, t_setup_);

  auto t1 = std::chrono::steady_clock::now();
  const int O = band_offsets(d, degree);
  for (int l = 0; l <= levels; ++l) {
    Level& L = levels_[l];
    if (l >= 1 && !host_assembly) continue;  // assembled on the device
    const std::int64_t S = L.mapper->lattice_size();
    L.band.assign(std::size_t(S) * O * K, 0.0);
    // patches in parallel, element chunks inside a patch in parallel
    const int outer = std::min(threads, K);
    const int inner = std::max(1, threads / outer);
    parallel_for(K, outer, [&](std::int64_t k) {
      assemble_patch_band(domain_->patches[k], degree, L.elements, L.band.data() + std::size_t(k) * O * S, inner);
    });
  }
  t_assemble_ = seconds_since(t1);

  auto t2 = std::chrono::steady_clock::now();
  {  // coarse matrix, summed global (multigrid.cpp:37-48, assembly.cpp:282-297)
    const Level& L0 = levels_[0];
    const int ext = L0.mapper->extent();
    const std::int64_t S = L0.mapper->lattice_size();
    const int N0 = int(L0.mapper->num_dofs());
    coarse_A_ = Dense(N0, N0);
    for (int k = 0; k < K; ++k) {
      const std::int32_t* l2g = L0.l2g.data() + k * S;
      const double* band = L0.band.data() + std::size_t(k) * O * S;
      for (std::int64_t r = 0; r < S; ++r) {
        if (l2g[r] < 0) continue;
        int ri[3] = {0, 0, 0};
        std::int64_t rem = r;
        for (int a = 0; a < d; ++a) {
          ri[a] = int(rem % ext);
          rem /= ext;
        }
        for (int o = 0; o < O; ++o) {
          int orem = o;
          std::int64_t c = 0, stride = 1;
          bool ok = true;
          for (int a = 0; a < d; ++a) {
            const int delta = orem % (2 * degree + 1) - degree;
            orem /= 2 * degree + 1;
            const int ca = ri[a] + delta;
            if (ca < 0 || ca >= ext) ok = false;
            c += std::int64_t(ca) * stride;
            stride *= ext;
          }
          if (!ok || l2g[c] < 0) continue;
          coarse_A_(l2g[r], l2g[c]) += band[std::size_t(o) * S + r];
        }
      }
    }
    try {
      coarse_L_ = N0 > 0 ? dense_cholesky(coarse_A_) : Dense();
    } catch (const DefinitenessError&) {
      throw DecompositionError("hierarchy: coarse factorization failed");
    }
  }
  t_setup_ += seconds_since(t2);
  if (timing) std::fprintf(stderr, "[pmg setup] coarse matrix + Cholesky %.2f s\n", seconds_since(t2));
  auto t3 = std::chrono::steady_clock::now();
  rhs_ = assemble_rhs(*levels_.back().mapper, rhs, threads);
  if (timing) std::fprintf(stderr, "[pmg setup] load vector %.2f s\n", seconds_since(t3));
}

// ============================================================ domains
namespace {

std::vector<int> parse_ints(const std::string& s) {
  std::vector<int> out;
  std::stringstream ss(s);
  std::string tok;
  while (std::getline(ss, tok, ',')) out.push_back(std::stoi(tok));
  return out;
}

using Tags = std::array<SideTag, 6>;

MultiPatchDomain boxes_2d(const std::vector<std::array<double, 4>>& boxes, const std::vector<Tags>& tags) {
  MultiPatchDomain d;
  d.dim = 2;
  for (const auto& b : boxes) d.patches.push_back(GeometryMap::axis_aligned_box({b[0], b[1]}, {b[2], b[3]}));
  d.side_tags = tags;
  build_topology(d);
  return d;
}

/// Structured kx x ky (x kz) grid of degree-1 single-element patches over a
/// vertex lattice with spacing w; `disp` perturbs every global vertex; sides on
/// the outer boundary get `tag_of(axis, end)`.
template <class Disp, class TagOf>
MultiPatchDomain vertex_grid(int dim, const int* k, double w, Disp&& disp, TagOf&& tag_of) {
  MultiPatchDomain dom;
  dom.dim = dim;
  const int nv[3] = {k[0] + 1, k[1] + 1, dim == 3 ? k[2] + 1 : 1};
  std::vector<std::array<double, 3>> vert(std::size_t(nv[0]) * nv[1] * nv[2]);
  for (int z = 0; z < nv[2]; ++z)
    for (int y = 0; y < nv[1]; ++y)
      for (int x = 0; x < nv[0]; ++x) {
        const int id = (z * nv[1] + y) * nv[0] + x;
        const int ix[3] = {x, y, z};
        std::array<double, 3> p{x * w, y * w, z * w};
        std::array<double, 3> dv{0.0, 0.0, 0.0};
        disp(id, p, dv);
        // a vertex on a boundary plane keeps that coordinate: boundary
        // vertices move tangentially only, so the outer shape is unchanged
        for (int a = 0; a < dim; ++a)
          if (ix[a] != 0 && ix[a] != k[a]) p[a] += dv[a];
        vert[id] = p;
      }
  const int pz = dim == 3 ? k[2] : 1;
  for (int cz = 0; cz < pz; ++cz)
    for (int cy = 0; cy < k[1]; ++cy)
      for (int cx = 0; cx < k[0]; ++cx) {
        std::vector<double> ctrl(std::size_t((1 << dim) * dim));
        for (int f = 0; f < (1 << dim); ++f) {
          const int vx = cx + (f & 1), vy = cy + ((f >> 1) & 1), vz = dim == 3 ? cz + ((f >> 2) & 1) : 0;
          const auto& v = vert[(vz * nv[1] + vy) * nv[0] + vx];
          for (int a = 0; a < dim; ++a) ctrl[f * dim + a] = v[a];
        }
        dom.patches.push_back(GeometryMap(std::vector<UnivariateSpace>(dim, UnivariateSpace(1, 1)), std::move(ctrl)));
        Tags t{};
        const int c[3] = {cx, cy, cz};
        for (int s = 0; s < 2 * dim; ++s) {
          const int a = side_axis(s), e = side_end(s);
          const bool outer = (e == 0 && c[a] == 0) || (e == 1 && c[a] == k[a] - 1);
          t[s] = outer ? tag_of(a, e) : SideTag::neumann;
        }
        dom.side_tags.push_back(t);
      }
  build_topology(dom);
  return dom;
}

}  // namespace

MultiPatchDomain make_domain(const std::string& spec, std::uint64_t seed) {
  const SideTag D = SideTag::dirichlet, N = SideTag::neumann;
  auto all = [](SideTag t) { return Tags{t, t, t, t, t, t}; };
  if (spec == "unit_square_D" || spec == "unit_square_N")
    return boxes_2d({{0, 0, 1, 1}}, {all(spec.back() == 'D' ? D : N)});
  if (spec == "two_squares_D" || spec == "two_squares_N") {
    const SideTag t = spec.back() == 'D' ? D : N;
    return boxes_2d({{0, 0, 1, 1}, {1, 0, 1, 1}}, {all(t), all(t)});
  }
  if (spec == "two_squares_flipped_D" || spec == "two_squares_flipped_N") {  // tests/util.hpp:58-73
    const SideTag t = spec.back() == 'D' ? D : N;
    MultiPatchDomain d;
    d.dim = 2;
    d.patches.push_back(GeometryMap::axis_aligned_box({0, 0}, {1, 1}));
    GeometryMap right = GeometryMap::axis_aligned_box({1, 0}, {1, 1});
    std::vector<double> c = right.control_points(), fl = c;
    for (int a = 0; a < 2; ++a) {
      fl[0 * 2 + a] = c[2 * 2 + a];
      fl[1 * 2 + a] = c[3 * 2 + a];
      fl[2 * 2 + a] = c[0 * 2 + a];
      fl[3 * 2 + a] = c[1 * 2 + a];
    }
    d.patches.push_back(GeometryMap(right.spaces(), fl));
    d.side_tags = {all(t), all(t)};
    build_topology(d);
    return d;
  }
  if (spec == "lshape")  // harness.cpp:142-155
    return boxes_2d({{0, 0, 1, 1}, {1, 0, 1, 1}, {0, 1, 1, 1}},
                    {Tags{D, N, D, N, N, N}, Tags{N, N, D, N, N, N}, Tags{D, N, N, N, N, N}});
  if (spec == "fichera") {  // harness.cpp:118-140
    MultiPatchDomain d;
    d.dim = 3;
    for (int cz = 0; cz < 2; ++cz)
      for (int cy = 0; cy < 2; ++cy)
        for (int cx = 0; cx < 2; ++cx) {
          if (cx == 1 && cy == 1 && cz == 1) continue;
          d.patches.push_back(GeometryMap::axis_aligned_box({double(cx), double(cy), double(cz)}, {1, 1, 1}));
          Tags t = all(N);
          const int c[3] = {cx, cy, cz};
          for (int a = 0; a < 3; ++a)
            if (c[a] == 0) t[side_of(a, 0)] = D;
          d.side_tags.push_back(t);
        }
    build_topology(d);
    return d;
  }
  if (spec.rfind("unit_grid(", 0) == 0 && spec.back() == ')') {  // harness.cpp:157-178
    std::vector<int> k = parse_ints(spec.substr(10, spec.size() - 11));
    if (k.size() < 2 || k.size() > 3) throw ConfigError("unit_grid: takes 2 or 3 patch counts");
    for (int v : k)
      if (v < 1) throw ConfigError("unit_grid: patch counts must be at least 1 per direction");
    MultiPatchDomain d;
    d.dim = int(k.size());
    const int kz = d.dim == 3 ? k[2] : 1;
    for (int z = 0; z < kz; ++z)
      for (int j = 0; j < k[1]; ++j)
        for (int i = 0; i < k[0]; ++i) {
          if (d.dim == 2)
            d.patches.push_back(GeometryMap::axis_aligned_box({double(i), double(j)}, {1, 1}));
          else
            d.patches.push_back(GeometryMap::axis_aligned_box({double(i), double(j), double(z)}, {1, 1, 1}));
          d.side_tags.push_back(all(D));
        }
    build_topology(d);
    return d;
  }
  // ---- BASELINE configs ----
  if (spec == "c1" || spec == "c3") {  // affine 2x2 / 4x4 split of the unit square, all Dirichlet
    const int k[3] = {spec == "c1" ? 2 : 4, spec == "c1" ? 2 : 4, 1};
    return vertex_grid(2, k, 1.0 / k[0], [](int, const std::array<double, 3>&, std::array<double, 3>&) {},
                       [&](int, int) { return D; });
  }
  if (spec == "c2") {  // 4x4, smooth sinusoidal vertex displacement of amplitude 0.05 w
    const int k[3] = {4, 4, 1};
    const double w = 0.25, A = 0.05 * w;
    const double ph1 = 2.0 * M_PI * unit_draw(seed, 1), ph2 = 2.0 * M_PI * unit_draw(seed, 2);
    return vertex_grid(
        2, k, w,
        [&](int, const std::array<double, 3>& p, std::array<double, 3>& dv) {
          dv[0] = A * std::sin(M_PI * p[0]) * std::sin(2.0 * M_PI * p[1] + ph1);
          dv[1] = A * std::sin(M_PI * p[1]) * std::sin(2.0 * M_PI * p[0] + ph2);
        },
        [&](int, int) { return D; });
  }
  auto jittered = [&](int kx, int ky, int kz, double w) {
    const int k[3] = {kx, ky, kz};
    return vertex_grid(
        3, k, w,
        [&](int id, const std::array<double, 3>&, std::array<double, 3>& dv) {
          for (int a = 0; a < 3; ++a) dv[a] = 0.05 * w * (2.0 * unit_draw(seed, 1000 + 3 * std::uint64_t(id) + a) - 1.0);
        },
        [&](int a, int) { return a == 0 ? D : N; });  // Dirichlet on x = min/max, Neumann elsewhere
  };
  if (spec == "c4") return jittered(2, 2, 2, 0.5);
  if (spec == "c5") return jittered(4, 4, 2, 1.0);
  if (spec.rfind("jitter(", 0) == 0 && spec.back() == ')') {  // weak-scaling boxes of unit cubes
    std::vector<int> k = parse_ints(spec.substr(7, spec.size() - 8));
    if (k.size() != 3) throw ConfigError("jitter: takes 3 patch counts");
    return jittered(k[0], k[1], k[2], 1.0);
  }
  throw ConfigError("domain: unknown descriptor '" + spec + "'");
}

}  // namespace pmg
