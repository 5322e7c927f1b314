// The reference's own solver templates driving the B200 backend -- TEST
// INFRASTRUCTURE (the drop-in check of include/patchmg_gpu_reference.hpp).
//
// This translation unit includes the reference's header
// /root/reference/proj/include/patchmg/multigrid.hpp as it lies (it is not
// copied into the repository; oracle/ref_templates/build.sh compiles this file
// against it, output in oracle/_ref/).  Eigen3 is absent from the image, so
// eigen_decl/ supplies declaration-only Eigen types for the header to parse;
// nothing Eigen is called.  It then runs
//   patchmg::pcg_generic(b, f, 1e-8, 500, precond, history)
// with precond = patchmg::mg_precondition(b, r) -- multigrid.hpp:120-189,
// unchanged -- over patchmg_gpu::ReferenceGpuBackend (every Backend method
// one call of libpmg_cuda's C ABI), next to the device-resident fused solve
// of the same context, and checks the reference's error behaviour through
// the backend (a level mismatch raises patchmg::DomainError, the iteration
// cap patchmg::DivergenceError).  Prints one JSON line.
//   pcg_ref_templates <domain> <degree> <levels> <n0>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <type_traits>
#include <vector>

#include "patchmg/multigrid.hpp"  // the reference (-I /root/reference/proj/include)
#include "patchmg_gpu_reference.hpp"
#include "pmg_host.h"

using Backend = patchmg_gpu::ReferenceGpuBackend;
static_assert(std::is_same_v<decltype(std::declval<const Backend&>().params()), const patchmg::CycleParams&>,
              "params() must bind the reference's CycleParams");

int main(int argc, char** argv) {
  const char* domain = argc > 1 ? argv[1] : "lshape";
  const int degree = argc > 2 ? std::atoi(argv[2]) : 2;
  const int levels = argc > 3 ? std::atoi(argv[3]) : 3;
  const int n0 = argc > 4 ? std::atoi(argv[4]) : 1;
  pmg_cycle_params prm{1, 1, 0.25, 0.2, 0};
  pmgh_hierarchy* h = nullptr;
  if (pmgh_build(domain, 1, degree, n0, levels, &prm, PMGH_RHS_DEFAULT, 42, 8, &h) != PMG_OK) {
    std::fprintf(stderr, "build: %s\n", pmgh_last_error());
    return 2;
  }
  pmg_hierarchy_desc desc;
  pmgh_describe(h, &desc);
  const double* rhs = nullptr;
  int64_t n = 0;
  pmgh_rhs(h, &rhs, &n);
  std::vector<double> f(rhs, rhs + n);
  int rc = 0;
  try {
    Backend b(desc, 0);
    const int L = b.finest_level();
    const Backend::DistVec fd = b.to_distributed_owner(L, f);
    std::vector<double> hist;
    const auto precond = [&](const Backend::DistVec& r) { return patchmg::mg_precondition(b, r); };
    const Backend::AccVec u = patchmg::pcg_generic(b, fd, 1e-8, 500, precond, hist);
    const std::vector<double> ug = b.gather_global(L, u, n);
    // the fused device solve on the same context
    std::vector<double> u2(size_t(n), 0.0), hist2(501, 0.0);
    int it2 = 0;
    patchmg_gpu::ReferenceErrors::raise(pmg_pcg_solve(b.ctx(), f.data(), n, 1e-8, 500, u2.data(), hist2.data(), &it2),
                                        pmg_last_error(b.ctx()));
    double diff = 0.0, scale = 0.0, hdiff = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      diff = std::max(diff, std::abs(ug[i] - u2[i]));
      scale = std::max(scale, std::abs(u2[i]));
    }
    // residual norms while ||r_k|| >= 1e-4 ||r_0|| (the tail carries the
    // O(eps ||r_0||) residual gap of two summation orders)
    for (size_t k = 0; k < hist.size() && int(k) <= it2; ++k)
      if (hist2[k] >= 1e-4 * hist2[0]) hdiff = std::max(hdiff, std::abs(hist[k] - hist2[k]) / hist2[k]);
    // error behaviour through the reference's exception classes
    bool domain_error = false, divergence_error = false;
    try {
      (void)b.residual(L, b.to_distributed_owner(L - 1, std::vector<double>(size_t(desc.levels[L - 1].num_dofs))), u);
    } catch (const patchmg::DomainError&) {
      domain_error = true;
    }
    try {
      std::vector<double> h3;
      (void)patchmg::pcg_generic(b, fd, 1e-8, 2, precond, h3);
    } catch (const patchmg::DivergenceError&) {
      divergence_error = true;
    }
    std::printf("{\"dofs\": %lld, \"template_iterations\": %d, \"fused_iterations\": %d, \"max_rel_diff\": %.3e, "
                "\"history_head_max_rel_diff\": %.3e, \"domain_error\": %s, \"divergence_error\": %s, \"u\": [",
                (long long)n, int(hist.size()) - 1, it2, diff / scale, hdiff, domain_error ? "true" : "false",
                divergence_error ? "true" : "false");
    for (int64_t i = 0; i < std::min<int64_t>(n, 8); ++i) std::printf("%s%.17g", i ? ", " : "", ug[i]);
    std::printf("]}\n");
  } catch (const patchmg::Error& e) {
    std::fprintf(stderr, "patchmg error: %s\n", e.what());
    rc = 1;
  }
  pmgh_free(h);
  return rc;
}
