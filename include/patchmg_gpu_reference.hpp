// patchmg_gpu_reference.hpp -- the GPU backend bound to the reference's own
// types, for a translation unit that already includes the reference's
// headers (/root/reference/proj/include/patchmg/multigrid.hpp).
//
//   #include "patchmg/multigrid.hpp"          // reference: CycleParams,
//   #include "patchmg_gpu_reference.hpp"      //   errors, the templates
//   patchmg_gpu::ReferenceGpuBackend b(desc);
//   auto u = patchmg::pcg_generic(b, f, tol, max_iter,
//       [&](const auto& r) { return patchmg::mg_precondition(b, r); }, history);
//
// params() returns `const patchmg::CycleParams&` (multigrid.hpp:21-27, the
// type mg_cycle_generic binds at multigrid.hpp:123) and every status code is
// rethrown as the reference's exception class (errors.hpp:9-56), so the
// reference's mg_cycle_generic / mg_precondition / pcg_generic
// (multigrid.hpp:120-189) compile and run against it unchanged.
#pragma once

#include "patchmg/errors.hpp"
#include "patchmg_gpu.hpp"

namespace patchmg_gpu {

struct ReferenceErrors {
  static void raise(int rc, const char* msg) {
    switch (rc) {
      case PMG_OK: return;
      case PMG_ERR_CONFIG: throw patchmg::ConfigError(msg);
      case PMG_ERR_DIVERGENCE: throw patchmg::DivergenceError(msg);
      case PMG_ERR_TRANSPORT: throw patchmg::TransportError(msg);
      case PMG_ERR_DOMAIN: throw patchmg::DomainError(msg);
      case PMG_ERR_DEFINITENESS: throw patchmg::DefinitenessError(msg);
      case PMG_ERR_DECOMPOSITION: throw patchmg::DecompositionError(msg);
      case PMG_ERR_GEOMETRY: throw patchmg::SingularGeometryError(msg);
      case PMG_ERR_NONMATCHING: throw patchmg::NonMatchingError(msg);
      default: throw patchmg::Error(msg);  // PMG_ERR_CUDA, PMG_ERR_GENERIC
    }
  }
};

using ReferenceGpuBackend = BasicGpuBackend<patchmg::CycleParams, ReferenceErrors>;

}  // namespace patchmg_gpu
