// extern "C" surface of the hierarchy builder (include/pmg_host.h).
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "../../../include/pmg_host.h"
#include "../common/rank_plan.hpp"
#include "hierarchy.hpp"

using namespace pmg;

struct pmgh_hierarchy {
  std::unique_ptr<Hierarchy> h;
  std::string domain;
  std::vector<pmg_level_desc> levels;
  std::vector<std::vector<pmg_piece_desc>> pieces;
  std::vector<std::vector<std::int32_t>> ts_start, ts_len, ts_off;
  std::vector<std::vector<double>> ts_vals;
  std::vector<std::int32_t> interfaces;
  std::vector<double> rhs;
  pmgplan::RankPlan plan;  // last pmgh_rank_plan result
  std::vector<std::int32_t> nb_rank, nb_off, nb_iface;
  std::vector<pmg_patch_geometry> geometry;  // empty if a patch map is not describable
  int flags = 0;                             // PMGH_* build flags
};

namespace {

thread_local std::string g_last_error;

int fail(int code, const char* what) {
  g_last_error = what;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    f();
    return PMG_OK;
  } catch (const ConfigError& e) {
    return fail(PMG_ERR_CONFIG, e.what());
  } catch (const DivergenceError& e) {
    return fail(PMG_ERR_DIVERGENCE, e.what());
  } catch (const TransportError& e) {
    return fail(PMG_ERR_TRANSPORT, e.what());
  } catch (const DomainError& e) {
    return fail(PMG_ERR_DOMAIN, e.what());
  } catch (const DefinitenessError& e) {
    return fail(PMG_ERR_DEFINITENESS, e.what());
  } catch (const DecompositionError& e) {
    return fail(PMG_ERR_DECOMPOSITION, e.what());
  } catch (const SingularGeometryError& e) {
    return fail(PMG_ERR_GEOMETRY, e.what());
  } catch (const NonMatchingError& e) {
    return fail(PMG_ERR_NONMATCHING, e.what());
  } catch (const NonManifoldError& e) {
    return fail(PMG_ERR_NONMATCHING, e.what());
  } catch (const std::exception& e) {
    return fail(PMG_ERR_GENERIC, e.what());
  }
}

int resolve_rhs_kind(const std::string& domain, int dim, int kind) {
  if (kind != PMGH_RHS_DEFAULT) return kind;
  if (domain == "c1") return PMGH_RHS_SINE_PI;
  if (domain.size() == 2 && domain[0] == 'c') return PMGH_RHS_RANDOM_NODES;
  if (domain.rfind("jitter(", 0) == 0) return PMGH_RHS_RANDOM_NODES;
  return dim == 2 ? PMGH_RHS_SINE2D : PMGH_RHS_SINE3D;
}

RhsSpec rhs_spec(const std::string& domain, int dim, int kind, std::uint64_t seed) {
  kind = resolve_rhs_kind(domain, dim, kind);
  RhsSpec s;
  s.seed = seed;
  switch (kind) {
    case PMGH_RHS_ONE:
      s.f = [](const double*) { return 1.0; };
      break;
    case PMGH_RHS_ZERO:
      s.f = [](const double*) { return 0.0; };
      s.zero = true;  // no quadrature loop: the load vector comes from elsewhere (pmg_assemble_load)
      break;
    case PMGH_RHS_SINE2D:  // harness.cpp:28-30
      s.f = [](const double* x) { return 50.0 * M_PI * M_PI * std::sin(5 * M_PI * x[0]) * std::sin(5 * M_PI * x[1]); };
      break;
    case PMGH_RHS_SINE3D:  // harness.cpp:32-35
      s.f = [](const double* x) {
        return 75.0 * M_PI * M_PI * std::sin(5 * M_PI * x[0]) * std::sin(5 * M_PI * x[1]) * std::sin(5 * M_PI * x[2]);
      };
      break;
    case PMGH_RHS_SINE_PI:
      s.f = [](const double* x) { return 2.0 * M_PI * M_PI * std::sin(M_PI * x[0]) * std::sin(M_PI * x[1]); };
      break;
    case PMGH_RHS_RANDOM_NODES:
      s.kind = RhsSpec::random_nodes;
      break;
    default:
      throw ConfigError("rhs: unknown source kind");
  }
  return s;
}

void fill_descriptors(pmgh_hierarchy* H) {
  const Hierarchy& h = *H->h;
  const int nl = h.num_levels();
  H->levels.assign(nl, pmg_level_desc{});
  H->pieces.assign(nl, {});
  H->ts_start.assign(nl, {});
  H->ts_len.assign(nl, {});
  H->ts_off.assign(nl, {});
  H->ts_vals.assign(nl, {});
  for (int l = 0; l < nl; ++l) {
    const Level& L = h.level(l);
    pmg_level_desc& d = H->levels[l];
    d.elements = L.elements;
    d.num_dofs = L.mapper->num_dofs();
    d.l2g = L.l2g.data();
    d.band_format = L.band.empty() ? PMG_BAND_ASSEMBLE : PMG_BAND_TENSOR;
    d.band = L.band.empty() ? nullptr : L.band.data();
    // matrix-free levels: the band (when assembled) stays available to host
    // consumers (the CPU checker); the CUDA context does not read it
    if ((H->flags & PMGH_KRONECKER) && l >= 1) d.band_format = PMG_BAND_KRONECKER;
    if (l >= 1) {
      const TwoScaleMatrix& P = L.two_scale;
      d.ts_fine_dim = P.fine_dim;
      d.ts_coarse_dim = P.coarse_dim;
      for (int i = 0; i < P.fine_dim; ++i) {
        H->ts_start[l].push_back(P.row_start[i]);
        H->ts_len[l].push_back(int(P.row_vals[i].size()));
        H->ts_off[l].push_back(int(H->ts_vals[l].size()));
        for (double v : P.row_vals[i]) H->ts_vals[l].push_back(v);
      }
      d.ts_row_start = H->ts_start[l].data();
      d.ts_row_len = H->ts_len[l].data();
      d.ts_row_off = H->ts_off[l].data();
      d.ts_vals = H->ts_vals[l].data();
    }
    auto& pv = H->pieces[l];
    pv.resize(L.pieces.size());
    for (std::size_t i = 0; i < L.pieces.size(); ++i) {
      const PieceData& src = L.pieces[i];
      pmg_piece_desc& p = pv[i];
      std::memset(&p, 0, sizeof p);
      p.kind = int(src.kind);
      p.patch = src.patch;
      p.ndofs = std::int64_t(src.dofs.size());
      p.dofs = src.dofs.data();
      if (src.kind == PieceKind::interior || src.kind == PieceKind::face) {
        p.naxes = src.fd.naxes;
        for (int a = 0; a < 3; ++a) {
          p.dims[a] = src.fd.dims[a];
          p.V[a] = a < src.fd.naxes ? src.fd.V[a]->data() : nullptr;
        }
        p.diag = src.fd.diag.data();
      } else if (src.kind == PieceKind::edge) {
        p.chol_dim = src.chol.dim();
        p.chol_bw = src.chol.bandwidth();
        p.chol_l = src.chol.factor().data();
      } else {
        p.scalar = src.scalar;
      }
    }
    d.num_pieces = int(pv.size());
    d.pieces = pv.data();
  }
  // patch geometry for device assembly: uniform open-knot spaces, free ends
  H->geometry.clear();
  for (const GeometryMap& g : h.domain().patches) {
    pmg_patch_geometry pg;
    std::memset(&pg, 0, sizeof pg);
    bool ok = true;
    for (int a = 0; a < g.dim(); ++a) {
      const UnivariateSpace& sp = g.spaces()[a];
      ok = ok && sp.left() == EndCondition::free_end && sp.right() == EndCondition::free_end;
      pg.degree[a] = sp.degree();
      pg.elements[a] = sp.elements();
    }
    pg.ctrl = g.control_points().data();
    if (!ok) {
      H->geometry.clear();
      break;
    }
    H->geometry.push_back(pg);
  }
  H->interfaces.clear();
  for (const auto& ifc : h.domain().interfaces) {
    H->interfaces.push_back(ifc.patch_a);
    H->interfaces.push_back(ifc.side_a);
    H->interfaces.push_back(ifc.patch_b);
    H->interfaces.push_back(ifc.side_b);
    H->interfaces.push_back(ifc.orientation);
  }
}

UnivariateSpace space_of(int degree, int elements, int le, int re) {
  return UnivariateSpace(degree, elements, le ? EndCondition::eliminated : EndCondition::free_end,
                         re ? EndCondition::eliminated : EndCondition::free_end);
}

}  // namespace

extern "C" {

const char* pmgh_last_error(void) { return g_last_error.c_str(); }

int pmgh_build(const char* domain, int split, int degree, int n0, int levels, const pmg_cycle_params* params,
               int rhs_kind, uint64_t seed, int threads, pmgh_hierarchy** out) {
  return pmgh_build_ex(domain, split, degree, n0, levels, params, rhs_kind, seed, threads, 0, out);
}

int pmgh_build_ex(const char* domain, int split, int degree, int n0, int levels, const pmg_cycle_params* params,
                  int rhs_kind, uint64_t seed, int threads, int flags, pmgh_hierarchy** out) {
  if (!out || !domain) return fail(PMG_ERR_CONFIG, "pmgh_build: null argument");
  *out = nullptr;
  return guarded([&] {
    auto H = std::make_unique<pmgh_hierarchy>();
    H->domain = domain;
    MultiPatchDomain dom = make_domain(domain, seed);
    if (split > 1) dom = split_patches(dom, split);
    CycleParams cp;
    if (params) {
      cp.nu = params->nu;
      cp.mu = params->mu;
      cp.tau = params->tau;
      cp.sigma_scale = params->sigma_scale;
      cp.damp_coarse = params->damp_coarse != 0;
    }
    RhsSpec rs = rhs_spec(H->domain, dom.dim, rhs_kind, seed);
    H->h = std::make_unique<Hierarchy>(dom, degree, n0, levels, cp, rs, threads,
                                       (flags & PMGH_DEVICE_ASSEMBLY) == 0);
    if ((flags & PMGH_DEVICE_ASSEMBLY) && dom.patches.empty()) throw ConfigError("pmgh_build: no patches");
    H->flags = flags;
    fill_descriptors(H.get());
    *out = H.release();
  });
}

void pmgh_free(pmgh_hierarchy* h) { delete h; }

int pmgh_resolve_rhs_kind(const char* domain, int dim, int rhs_kind) {
  return resolve_rhs_kind(domain ? domain : "", dim, rhs_kind);
}

int pmgh_describe(pmgh_hierarchy* H, pmg_hierarchy_desc* out) {
  if (!H || !out) return fail(PMG_ERR_CONFIG, "pmgh_describe: null argument");
  const Hierarchy& h = *H->h;
  out->dim = h.dim();
  out->degree = h.degree();
  out->num_patches = h.num_patches();
  out->num_levels = h.num_levels();
  out->params.nu = h.params().nu;
  out->params.mu = h.params().mu;
  out->params.tau = h.params().tau;
  out->params.sigma_scale = h.params().sigma_scale;
  out->params.damp_coarse = h.params().damp_coarse ? 1 : 0;
  out->levels = H->levels.data();
  out->coarse_n = h.coarse_matrix().rows;
  out->coarse_A = h.coarse_matrix().data();
  out->coarse_L = h.coarse_factor().data();
  out->geometry = H->geometry.empty() ? nullptr : H->geometry.data();
  return PMG_OK;
}

int pmgh_rhs(pmgh_hierarchy* H, const double** rhs, int64_t* n) {
  if (!H || !rhs || !n) return fail(PMG_ERR_CONFIG, "pmgh_rhs: null argument");
  const std::vector<double>& r = H->rhs.empty() ? H->h->rhs() : H->rhs;
  *rhs = r.data();
  *n = std::int64_t(r.size());
  return PMG_OK;
}

int pmgh_set_rhs(pmgh_hierarchy* H, int rhs_kind, uint64_t seed, int threads) {
  if (!H) return fail(PMG_ERR_CONFIG, "pmgh_set_rhs: null argument");
  return guarded([&] {
    const Hierarchy& h = *H->h;
    RhsSpec rs = rhs_spec(H->domain, h.dim(), rhs_kind, seed);
    H->rhs = assemble_rhs(*h.level(h.finest_level()).mapper, rs, threads);
  });
}

double pmgh_seconds(pmgh_hierarchy* H, int which) {
  if (!H) return -1.0;
  return which == 0 ? H->h->setup_seconds() : H->h->assemble_seconds();
}

int64_t pmgh_stored_entries(int degree, int elements, int dim, int patches) {
  return stored_stiffness_entries(degree, elements, dim, patches);
}

int pmgh_reps(pmgh_hierarchy* H, int level, const int32_t** off, const int32_t** patch, const int32_t** local) {
  if (!H || level < 0 || level >= H->h->num_levels()) return fail(PMG_ERR_CONFIG, "pmgh_reps: bad level");
  const DofMapper& m = *H->h->level(level).mapper;
  *off = m.rep_offsets().data();
  *patch = m.rep_patches().data();
  *local = m.rep_locals().data();
  return PMG_OK;
}

int pmgh_interfaces(pmgh_hierarchy* H, int* count, const int32_t** data) {
  if (!H || !count || !data) return fail(PMG_ERR_CONFIG, "pmgh_interfaces: null argument");
  *count = int(H->interfaces.size() / 5);
  *data = H->interfaces.data();
  return PMG_OK;
}

int pmgh_rank_plan(pmgh_hierarchy* H, int level, int ranks, int rank, pmgh_rank_plan_view* out) {
  if (!H || !out || level < 0 || level >= H->h->num_levels()) return fail(PMG_ERR_CONFIG, "pmgh_rank_plan: bad args");
  return guarded([&] {
    const Level& L = H->h->level(level);
    pmgplan::Partition part;
    try {
      part = pmgplan::contiguous(H->h->num_patches(), ranks);
    } catch (const std::invalid_argument& e) {
      throw ConfigError(e.what());
    }
    if (rank < 0 || rank >= ranks) throw ConfigError("pmgh_rank_plan: rank out of range");
    H->plan = pmgplan::build(L.l2g.data(), H->h->num_patches(), L.mapper->lattice_size(), L.mapper->num_dofs(), part,
                             rank);
    H->nb_rank.clear();
    H->nb_off.assign(1, 0);
    H->nb_iface.clear();
    for (const auto& nb : H->plan.neighbors) {
      H->nb_rank.push_back(nb.rank);
      H->nb_iface.insert(H->nb_iface.end(), nb.iface.begin(), nb.iface.end());
      H->nb_off.push_back(int(H->nb_iface.size()));
    }
    out->n_iface = int(H->plan.iface_g.size());
    out->iface_g = H->plan.iface_g.data();
    out->rep_off = H->plan.rep_off.data();
    out->rep_slot = H->plan.rep_slot.data();
    out->comb_off = H->plan.comb_off.data();
    out->comb_src = H->plan.comb_src.data();
    out->n_neighbors = int(H->nb_rank.size());
    out->nb_rank = H->nb_rank.data();
    out->nb_off = H->nb_off.data();
    out->nb_iface = H->nb_iface.data();
  });
}

int pmgh_gauss_legendre(int points, double* nodes, double* weights) {
  return guarded([&] {
    const QuadratureRule& r = gauss_legendre(points);
    for (int i = 0; i < points; ++i) {
      nodes[i] = r.nodes[i];
      weights[i] = r.weights[i];
    }
  });
}

int pmgh_eval_basis(int degree, int elements, int le, int re, double x, int deriv, int* first_index, double* values) {
  return guarded([&] {
    BasisEval b = eval_basis(space_of(degree, elements, le, re), x, deriv);
    *first_index = b.first_index;
    for (int i = 0; i <= degree; ++i) values[i] = b.values[i];
  });
}

int pmgh_gram(int degree, int elements, int le, int re, int deriv, int* dim, double* out) {
  return guarded([&] {
    UnivariateSpace s = space_of(degree, elements, le, re);
    *dim = s.dimension();
    if (!out) return;
    Dense m = (deriv ? univariate_stiffness(s) : univariate_mass(s)).to_dense();
    std::memcpy(out, m.data(), sizeof(double) * m.a.size());
  });
}

int pmgh_two_scale(int degree, int elements, int le, int re, int* fine_dim, int* coarse_dim, double* dense) {
  return guarded([&] {
    TwoScaleMatrix P = two_scale_matrix(space_of(degree, elements, le, re));
    *fine_dim = P.fine_dim;
    *coarse_dim = P.coarse_dim;
    if (!dense) return;
    Dense m = P.to_dense();
    std::memcpy(dense, m.data(), sizeof(double) * m.a.size());
  });
}

int pmgh_gen_eig(int n, const double* K, const double* M, double* eigenvalues, double* eigenvectors) {
  return guarded([&] {
    Dense k(n, n), m(n, n);
    std::memcpy(k.data(), K, sizeof(double) * n * n);
    std::memcpy(m.data(), M, sizeof(double) * n * n);
    GenEigDecomposition g = gen_eig(k, m);
    std::memcpy(eigenvalues, g.eigenvalues.data(), sizeof(double) * n);
    std::memcpy(eigenvectors, g.eigenvectors.data(), sizeof(double) * n * n);
  });
}

int pmgh_banded_cholesky_solve(int dim, int bw, const double* lower_band, const double* rhs, double* x) {
  return guarded([&] {
    BandedSymMatrix a(dim, bw);
    for (int i = 0; i < dim; ++i)
      for (int k = 0; k <= bw && k <= i; ++k) a.add(i, i - k, lower_band[std::size_t(i) * (bw + 1) + k]);
    BandedCholesky c(a);
    c.solve(rhs, x);
  });
}

}  // extern "C"
