"""Hierarchy: the multigrid setup the solve path consumes, built on the host by
libpmg_host.so -- the counterpart of patchmg::Hierarchy
(include/patchmg/multigrid.hpp:42-75, src/multigrid.cpp:16-50) plus the
load vector (assemble_rhs, src/assembly.cpp:299-365)."""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

from . import _native as N
from .errors import raise_for

RHS_KINDS = {"default": 0, "one": 1, "sine2d": 2, "sine3d": 3, "sine_pi": 4, "random_nodes": 5, "zero": 6}


@dataclass
class CycleParams:
    """multigrid.hpp:21-27"""
    nu: int = 1
    mu: int = 1
    tau: float = 0.25
    sigma_scale: float = 0.2
    damp_coarse: bool = False

    def to_c(self) -> N.PmgCycleParams:
        return N.PmgCycleParams(self.nu, self.mu, self.tau, self.sigma_scale, 1 if self.damp_coarse else 0)


class Hierarchy:
    """Levels 0..levels with n0 * 2**l elements per patch direction.

    assembly="device" leaves the stiffness of levels >= 1 unassembled on the
    host: a GpuBackend context assembles it on the B200 from the patch
    geometry (PMG_BAND_ASSEMBLE).  Such a hierarchy has no host band to give
    the oracle; tests pair it with a host-assembled twin.

    operator="kronecker" describes levels >= 1 as PMG_BAND_KRONECKER: the
    context applies the patch operator matrix-free as a Kronecker sum of
    univariate matrices (axis-aligned affine patch maps only: c1, c3,
    unit_grid, lshape, fichera ...).  The host band stays available to the
    oracle."""

    def __init__(self, domain: str, degree: int, levels: int, n0: int = 1, split: int = 1,
                 params: CycleParams | None = None, rhs: str = "default", seed: int = 42,
                 threads: int | None = None, assembly: str = "host", operator: str = "band"):
        if assembly not in ("host", "device"):
            raise ValueError("assembly must be 'host' or 'device'")
        if operator not in ("band", "kronecker"):
            raise ValueError("operator must be 'band' or 'kronecker'")
        self.assembly = assembly
        self.operator = operator
        lib = N.host_lib()
        self.params = params or CycleParams()
        self.domain = domain
        self.seed = seed
        self.threads = threads or os.cpu_count() or 1
        h = C.c_void_p()
        flags = (N.PMGH_DEVICE_ASSEMBLY if assembly == "device" else 0) | (
            N.PMGH_KRONECKER if operator == "kronecker" else 0)
        rc = lib.pmgh_build_ex(domain.encode(), split, degree, n0, levels, C.byref(self.params.to_c()),
                               RHS_KINDS[rhs], seed, self.threads, flags, C.byref(h))
        raise_for(rc, lib.pmgh_last_error().decode())
        self._h = h
        self.desc = N.PmgHierarchyDesc()
        raise_for(lib.pmgh_describe(h, C.byref(self.desc)), lib.pmgh_last_error().decode())

    # ---- shape
    @property
    def dim(self) -> int:
        return self.desc.dim

    @property
    def degree(self) -> int:
        return self.desc.degree

    @property
    def num_patches(self) -> int:
        return self.desc.num_patches

    @property
    def num_levels(self) -> int:
        return self.desc.num_levels

    @property
    def finest_level(self) -> int:
        return self.desc.num_levels - 1

    def elements(self, level: int) -> int:
        return self.desc.levels[level].elements

    def extent(self, level: int) -> int:
        return self.elements(level) + self.degree

    def lattice_size(self, level: int) -> int:
        return self.extent(level) ** self.dim

    def num_dofs(self, level: int) -> int:
        return int(self.desc.levels[level].num_dofs)

    def stored_entries(self, level: int) -> int:
        """Stored CSR entries of the reference layout (harness.cpp:274-282)."""
        return int(N.host_lib().pmgh_stored_entries(self.degree, self.elements(level), self.dim, self.num_patches))

    # ---- data views (valid while self lives)
    def l2g(self, level: int) -> np.ndarray:
        n = self.num_patches * self.lattice_size(level)
        return np.ctypeslib.as_array(self.desc.levels[level].l2g, shape=(n,)).reshape(self.num_patches, -1)

    def band(self, level: int) -> np.ndarray:
        if self.desc.levels[level].band_format not in (N.PMG_BAND_TENSOR, N.PMG_BAND_KRONECKER) or not \
                self.desc.levels[level].band:
            raise ValueError(f"level {level} is assembled on the device; no host band")
        o = (2 * self.degree + 1) ** self.dim
        s = self.lattice_size(level)
        return np.ctypeslib.as_array(self.desc.levels[level].band, shape=(self.num_patches * o * s,)).reshape(
            self.num_patches, o, s)

    def adopt_device_bands(self, backend) -> float:
        """Give the levels assembled on the device (PMG_BAND_ASSEMBLE) host bands
        downloaded from `backend` (a single-GPU GpuBackend built on this
        hierarchy), so host consumers -- the CPU oracle and baseline -- read
        exactly the operator the device applies.  Returns seconds spent."""
        import time
        t = time.perf_counter()
        self._adopted = getattr(self, "_adopted", {})
        for level in range(self.num_levels):
            ld = self.desc.levels[level]
            if ld.band_format != N.PMG_BAND_ASSEMBLE:
                continue
            band = np.ascontiguousarray(backend.download_band(level))
            self._adopted[level] = band
            ld.band = band.ctypes.data_as(N._dp)
            ld.band_format = N.PMG_BAND_TENSOR
        self.assembly = "device (bands downloaded to the host)"
        return time.perf_counter() - t

    def pieces(self, level: int):
        ld = self.desc.levels[level]
        return [ld.pieces[i] for i in range(ld.num_pieces)]

    def coarse_matrix(self) -> np.ndarray:
        n = self.desc.coarse_n
        return np.ctypeslib.as_array(self.desc.coarse_A, shape=(n * n,)).reshape(n, n).T.copy()

    def two_scale_dense(self, level: int) -> np.ndarray:
        ld = self.desc.levels[level]
        P = np.zeros((ld.ts_fine_dim, ld.ts_coarse_dim))
        for i in range(ld.ts_fine_dim):
            for q in range(ld.ts_row_len[i]):
                P[i, ld.ts_row_start[i] + q] = ld.ts_vals[ld.ts_row_off[i] + q]
        return P

    def reps(self, level: int):
        off, pat, loc = N._ip(), N._ip(), N._ip()
        lib = N.host_lib()
        raise_for(lib.pmgh_reps(self._h, level, C.byref(off), C.byref(pat), C.byref(loc)), lib.pmgh_last_error().decode())
        nd = self.num_dofs(level)
        o = np.ctypeslib.as_array(off, shape=(nd + 1,)).copy()
        tot = int(o[-1])
        return o, np.ctypeslib.as_array(pat, shape=(tot,)).copy(), np.ctypeslib.as_array(loc, shape=(tot,)).copy()

    def interfaces(self):
        cnt, data = C.c_int(), N._ip()
        N.host_lib().pmgh_interfaces(self._h, C.byref(cnt), C.byref(data))
        if cnt.value == 0:
            return np.zeros((0, 5), dtype=np.int32)
        return np.ctypeslib.as_array(data, shape=(cnt.value * 5,)).reshape(-1, 5).copy()

    def rhs(self) -> np.ndarray:
        ptr, n = N._dp(), C.c_int64()
        N.host_lib().pmgh_rhs(self._h, C.byref(ptr), C.byref(n))
        return np.ctypeslib.as_array(ptr, shape=(n.value,)).copy()

    def set_rhs(self, kind: str, seed: int | None = None):
        lib = N.host_lib()
        raise_for(lib.pmgh_set_rhs(self._h, RHS_KINDS[kind], self.seed if seed is None else seed, self.threads),
                  lib.pmgh_last_error().decode())

    def setup_seconds(self) -> float:
        return N.host_lib().pmgh_seconds(self._h, 0)

    def assemble_seconds(self) -> float:
        return N.host_lib().pmgh_seconds(self._h, 1)

    def close(self):
        if getattr(self, "_h", None):
            N.host_lib().pmgh_free(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---- BASELINE.json configs: (domain, degree, n0, levels)
CONFIGS = {
    "c1": ("c1", 2, 2, 5),   # 2D 2x2 affine, p=2, 2 -> 64 elements per patch
    "c2": ("c2", 4, 2, 7),   # 2D 4x4 perturbed, p=4, 2 -> 256
    "c3p2": ("c3", 2, 2, 6), "c3p3": ("c3", 3, 2, 6), "c3p4": ("c3", 4, 2, 6),
    "c3p6": ("c3", 6, 2, 6), "c3p8": ("c3", 8, 2, 6),  # 2D 4x4 affine, 2 -> 128
    "c4": ("c4", 3, 2, 5),   # 3D 2x2x2 jittered, p=3, 2 -> 64
    "c5": ("c5", 3, 2, 5),   # 3D 4x4x2 jittered, p=3, 2 -> 64
}


def baseline_hierarchy(name: str, levels: int | None = None, seed: int = 42, threads: int | None = None) -> Hierarchy:
    """One of the BASELINE configs; `levels` overrides the refinement depth
    (smaller levels give the same problem family at desk scale)."""
    dom, p, n0, lv = CONFIGS[name]
    return Hierarchy(dom, p, lv if levels is None else levels, n0=n0, seed=seed, threads=threads)
