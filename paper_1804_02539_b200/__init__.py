"""B200-native (sm_100a) solve path of the Hofer-Takacs parallel multi-patch
IgA multigrid method (arXiv 1804.02539): PCG preconditioned by one V(1,1)
cycle with the subspace-corrected fast-diagonalization smoother.

  Hierarchy   host-side setup (libpmg_host.so)
  GpuBackend  the reference Backend concept over libpmg_cuda.so
"""
from .errors import (ConfigError, DecompositionError, DefinitenessError, DivergenceError, DomainError, Error,
                     NonMatchingError, SingularGeometryError, TransportError)
from .hierarchy import CONFIGS, CycleParams, Hierarchy, baseline_hierarchy

__all__ = [
    "Hierarchy", "CycleParams", "CONFIGS", "baseline_hierarchy", "Error", "ConfigError", "DomainError",
    "DefinitenessError", "DivergenceError", "DecompositionError", "SingularGeometryError", "NonMatchingError",
    "TransportError",
]


def __getattr__(name):
    if name in ("GpuBackend", "AccVec", "DistVec", "SolveReport", "mg_cycle_generic", "mg_precondition",
                "pcg_generic"):
        from . import backend
        return getattr(backend, name)
    raise AttributeError(name)
