// C++ drop-in demonstration without the reference's headers: the restated
// pcg_generic / mg_precondition templates (include/patchmg_gpu.hpp, namespace
// patchmg_gpu::generic) driving GpuBackend through
// the C ABI, next to the device-resident fused solve.  Prints one JSON line.
//   pcg_cpp <domain> <degree> <levels> <n0>
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../../include/patchmg_gpu.hpp"
#include "../../../include/pmg_host.h"

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
  try {
    patchmg_gpu::GpuBackend b(desc, 0);
    const int L = b.finest_level();
    auto fd = b.to_distributed_owner(L, f);
    std::vector<double> hist;
    auto u = patchmg_gpu::generic::pcg_generic(
        b, fd, 1e-8, 500, [&](const patchmg_gpu::GpuBackend::DistVec& r) { return patchmg_gpu::generic::mg_precondition(b, r); },
        hist);
    std::vector<double> ug = b.gather_global(L, u, n);
    std::vector<double> u2(size_t(n), 0.0), hist2(501, 0.0);
    int it2 = 0;
    patchmg_gpu::check(pmg_pcg_solve(b.ctx(), f.data(), n, 1e-8, 500, u2.data(), hist2.data(), &it2),
                       pmg_last_error(b.ctx()));
    double diff = 0.0, scale = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      diff = std::max(diff, std::abs(ug[i] - u2[i]));
      scale = std::max(scale, std::abs(u2[i]));
    }
    std::printf("{\"dofs\": %lld, \"template_iterations\": %d, \"fused_iterations\": %d, \"max_rel_diff\": %.3e, "
                "\"u\": [",
                (long long)n, int(hist.size()) - 1, it2, diff / scale);
    for (int64_t i = 0; i < std::min<int64_t>(n, 8); ++i) std::printf("%s%.17g", i ? ", " : "", ug[i]);
    std::printf("]}\n");
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    pmgh_free(h);
    return 1;
  }
  pmgh_free(h);
  return 0;
}
