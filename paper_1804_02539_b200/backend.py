"""GpuBackend: the reference's Backend concept (SerialBackend,
include/patchmg/multigrid.hpp:80-114; ParallelBackend, parallel.hpp:267-341)
over the sm_100a C ABI of include/pmg_cuda.h, plus the solver templates
mg_cycle_generic / mg_precondition / pcg_generic (multigrid.hpp:120-189)
written once for any backend.

AccVec / DistVec are distinct handle types, as in the reference
(parallel.hpp:169-260); operations accept exactly the forms the reference's
signatures name.  There is no CPU path: a missing libpmg_cuda.so raises.
"""
from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from .errors import DefinitenessError, DivergenceError, DomainError, raise_for
from .hierarchy import CycleParams, Hierarchy


class _Vec:
    form = -1

    def __init__(self, backend: "GpuBackend", level: int):
        self._b = backend
        self.level = level
        h = C.c_void_p()
        backend._check(backend._lib.pmg_vec_create(backend._ctx, level, C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if self._h:
                self._b._lib.pmg_vec_free(self._h)
                self._h = None
        except Exception:
            pass

    def lattice(self) -> np.ndarray:
        """Raw per-patch lattice values (patches x (n+p)^d)."""
        n = self._b.lattice_size(self.level)
        out = np.empty(n)
        self._b._check(self._b._lib.pmg_vec_lattice_download(self._b._ctx, self._h, out.ctypes.data_as(N._dp), n))
        return out


class AccVec(_Vec):
    """Accumulated form: every replica holds the global value."""
    form = 0


class DistVec(_Vec):
    """Distributed form: the replicas' values sum to the global value."""
    form = 1


def _need(v, cls, level):
    if not isinstance(v, cls):
        raise TypeError(f"expected {cls.__name__}, got {type(v).__name__}")
    if v.level != level:
        raise DomainError(f"vector level {v.level} != {level}")


class GpuBackend:
    """One rank's backend.  comm=None: a single GPU owning every patch;
    otherwise a PmgCommDesc (see parallel.py) placing this context on its
    contiguous patch block with an NCCL or in-process-hub transport."""

    def __init__(self, hierarchy: Hierarchy, device: int = 0, comm: N.PmgCommDesc | None = None):
        self._lib = N.cuda_lib()
        self.h = hierarchy
        self.comm = comm
        self.rank = comm.rank if comm is not None else 0
        self.size = comm.size if comm is not None else 1
        ctx = C.c_void_p()
        rc = self._lib.pmg_ctx_create(C.byref(hierarchy.desc), device, C.byref(comm) if comm is not None else None,
                                      C.byref(ctx))
        raise_for(rc, self._lib.pmg_last_error(None).decode())
        self._ctx = ctx

    def comm_bytes(self) -> int:
        n = C.c_uint64()
        self._check(self._lib.pmg_comm_bytes(self._ctx, C.byref(n)))
        return n.value

    def close(self):
        if getattr(self, "_ctx", None):
            self._lib.pmg_ctx_destroy(self._ctx)
            self._ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int):
        if rc != 0:
            raise_for(rc, self._lib.pmg_last_error(self._ctx).decode())

    # ---- Backend concept
    def params(self) -> CycleParams:
        return self.h.params

    def finest_level(self) -> int:
        return self.h.finest_level

    def assembly_seconds(self) -> float:
        """Wall time of device stiffness assembly at context creation (0 if none)."""
        n = C.c_int64()
        self._check(self._lib.pmg_ctx_info(self._ctx, 5, C.byref(n)))
        return n.value / 1e6

    def load_seconds(self) -> float:
        """Wall time spent in assemble_load (device load-vector assembly)."""
        n = C.c_int64()
        self._check(self._lib.pmg_ctx_info(self._ctx, 7, C.byref(n)))
        return n.value / 1e6

    def assemble_load(self, rhs: str = "default", seed: int | None = None) -> DistVec:
        """The finest-level load vector assembled on the device from the patch
        geometry (pmg_assemble_load; assemble_rhs, assembly.cpp:299-365) as a
        DistributedVector.  rhs = a source name of Hierarchy (\"default\": the
        domain's own); seed defaults to the hierarchy's."""
        from .hierarchy import RHS_KINDS
        kind = N.host_lib().pmgh_resolve_rhs_kind(self.h.domain.encode(), self.h.dim, RHS_KINDS[rhs])
        v = DistVec(self, self.h.finest_level)
        self._check(self._lib.pmg_assemble_load(self._ctx, kind, self.h.seed if seed is None else seed, v._h))
        return v

    def download_band(self, level: int) -> np.ndarray:
        """The level's operator as held on the device, as the reference's
        index-free full band [K_local][(2p+1)^d][(n+p)^d] (pmg_band_download)."""
        h = self.h
        k = (self.h.num_patches if self.comm is None else self.comm.patch_end - self.comm.patch_begin)
        n = k * (2 * h.degree + 1) ** h.dim * h.lattice_size(level)
        out = np.empty(n)
        self._check(self._lib.pmg_band_download(self._ctx, level, out.ctypes.data_as(N._dp), n))
        return out.reshape(k, (2 * h.degree + 1) ** h.dim, h.lattice_size(level))

    def lattice_size(self, level: int) -> int:
        n = C.c_int64()
        self._check(self._lib.pmg_ctx_info(self._ctx, (level << 8) | 1, C.byref(n)))
        return n.value

    def zero_acc(self, level: int) -> AccVec:
        return AccVec(self, level)

    def zero_dist(self, level: int) -> DistVec:
        return DistVec(self, level)

    def apply_op(self, level: int, u: AccVec) -> DistVec:
        _need(u, AccVec, level)
        out = DistVec(self, level)
        self._check(self._lib.pmg_apply_op(self._ctx, level, u._h, out._h))
        return out

    def residual(self, level: int, f: DistVec, u: AccVec) -> DistVec:
        _need(f, DistVec, level)
        _need(u, AccVec, level)
        out = DistVec(self, level)
        self._check(self._lib.pmg_residual(self._ctx, level, f._h, u._h, out._h))
        return out

    def accumulate(self, level: int, r: DistVec) -> AccVec:
        _need(r, DistVec, level)
        out = AccVec(self, level)
        self._check(self._lib.pmg_accumulate(self._ctx, level, r._h, out._h))
        return out

    def smooth(self, level: int, r: DistVec) -> AccVec:
        _need(r, DistVec, level)
        out = AccVec(self, level)
        self._check(self._lib.pmg_smooth(self._ctx, level, r._h, out._h))
        return out

    def restrict_residual(self, level: int, r: DistVec) -> DistVec:
        _need(r, DistVec, level)
        out = DistVec(self, level - 1)
        self._check(self._lib.pmg_restrict(self._ctx, level, r._h, out._h))
        return out

    def add_prolonged(self, level: int, coarse: AccVec, c: float, u: AccVec) -> None:
        _need(coarse, AccVec, level - 1)
        _need(u, AccVec, level)
        self._check(self._lib.pmg_add_prolonged(self._ctx, level, coarse._h, c, u._h))

    def coarse_solve(self, r: DistVec) -> AccVec:
        _need(r, DistVec, 0)
        out = AccVec(self, 0)
        self._check(self._lib.pmg_coarse_solve(self._ctx, r._h, out._h))
        return out

    def dot(self, level: int, a: DistVec, b: AccVec) -> float:
        if isinstance(a, AccVec) and isinstance(b, DistVec):
            a, b = b, a
        _need(a, DistVec, level)
        _need(b, AccVec, level)
        out = C.c_double()
        self._check(self._lib.pmg_dot(self._ctx, level, a._h, b._h, C.byref(out)))
        return out.value

    def axpy_acc(self, a: float, x: AccVec, y: AccVec) -> None:
        _need(x, AccVec, y.level)
        _need(y, AccVec, x.level)
        self._check(self._lib.pmg_axpy(self._ctx, a, x._h, y._h))

    def axpy_dist(self, a: float, x: DistVec, y: DistVec) -> None:
        _need(x, DistVec, y.level)
        _need(y, DistVec, x.level)
        self._check(self._lib.pmg_axpy(self._ctx, a, x._h, y._h))

    def xpay_acc(self, z: AccVec, beta: float, p: AccVec) -> None:
        _need(z, AccVec, p.level)
        _need(p, AccVec, z.level)
        self._check(self._lib.pmg_xpay(self._ctx, z._h, beta, p._h))

    def copy(self, v):
        out = type(v)(self, v.level)
        self._check(self._lib.pmg_vec_copy(self._ctx, v._h, out._h))
        return out

    # ---- conversions (parallel.cpp:428-468)
    def to_accumulated(self, level: int, g: np.ndarray) -> AccVec:
        v = AccVec(self, level)
        g = np.ascontiguousarray(g, dtype=np.float64)
        self._check(self._lib.pmg_vec_upload(self._ctx, v._h, 0, g.ctypes.data_as(N._dp), g.size))
        return v

    def to_distributed_owner(self, level: int, g: np.ndarray) -> DistVec:
        v = DistVec(self, level)
        g = np.ascontiguousarray(g, dtype=np.float64)
        self._check(self._lib.pmg_vec_upload(self._ctx, v._h, 1, g.ctypes.data_as(N._dp), g.size))
        return v

    def gather_global(self, level: int, v) -> np.ndarray:
        """Accumulated: owner-replica values; distributed: replica sums."""
        out = np.empty(self.h.num_dofs(level))
        self._check(self._lib.pmg_vec_download(self._ctx, v._h, v.form, out.ctypes.data_as(N._dp), out.size))
        return out

    # ---- fused device paths
    def mg_cycle(self, level: int, u: AccVec, f: DistVec) -> None:
        _need(u, AccVec, level)
        _need(f, DistVec, level)
        self._check(self._lib.pmg_mg_cycle(self._ctx, level, u._h, f._h))

    def precondition(self, r: DistVec, out: AccVec | None = None) -> AccVec:
        """mg_precondition (multigrid.hpp:144-149); `out` reuses a vector (the
        library replays one cached graph per (r, z) pair)."""
        _need(r, DistVec, self.finest_level())
        z = AccVec(self, r.level) if out is None else out
        _need(z, AccVec, r.level)
        self._check(self._lib.pmg_precondition(self._ctx, r._h, z._h))
        return z

    def pcg_solve(self, f_global: np.ndarray, tol: float = 1e-8, max_iter: int = 500):
        """pcg_solve (multigrid.hpp:196-197) end to end from host memory."""
        f = np.ascontiguousarray(f_global, dtype=np.float64)
        u = np.empty_like(f)
        hist = np.zeros(max_iter + 1)
        it = C.c_int(0)
        rc = self._lib.pmg_pcg_solve(self._ctx, f.ctypes.data_as(N._dp), f.size, tol, max_iter,
                                     u.ctypes.data_as(N._dp), hist.ctypes.data_as(N._dp), C.byref(it))
        self._check(rc)
        return u, SolveReport(it.value, list(hist[: it.value + 1]))

    def pcg_solve_device(self, f: DistVec, tol: float = 1e-8, max_iter: int = 500, u: AccVec | None = None):
        if u is None:
            u = AccVec(self, f.level)
        hist = np.zeros(max_iter + 1)
        it = C.c_int(0)
        self._check(self._lib.pmg_pcg_solve_device(self._ctx, f._h, tol, max_iter, u._h,
                                                   hist.ctypes.data_as(N._dp), C.byref(it)))
        return u, SolveReport(it.value, list(hist[: it.value + 1]))

    def set_stream(self, stream_handle: int):
        self._check(self._lib.pmg_set_stream(self._ctx, C.c_void_p(stream_handle)))

    def synchronize(self):
        self._check(self._lib.pmg_synchronize(self._ctx))

    def kernel_launches(self, reset: bool = False) -> int:
        n = C.c_int64()
        self._check(self._lib.pmg_kernel_stats(self._ctx, 0, C.byref(n), None))
        if reset:
            self._check(self._lib.pmg_kernel_stats(self._ctx, 2, C.byref(C.c_int64()), None))
        return n.value


@dataclass
class SolveReport:
    """multigrid.hpp:29-35"""
    iterations: int = 0
    residual_history: list = field(default_factory=list)
    t_setup: float = 0.0
    t_assemble: float = 0.0
    t_solve: float = 0.0


# ---------------------------------------------------------------- templates
def mg_cycle_generic(b, level: int, u, f) -> None:
    """multigrid.hpp:120-141"""
    prm = b.params()
    for _ in range(prm.nu):
        z = b.smooth(level, b.residual(level, f, u))
        b.axpy_acc(prm.tau, z, u)
    rc = b.restrict_residual(level, b.residual(level, f, u))
    if level == 1:
        p = b.coarse_solve(rc)
    else:
        p = b.zero_acc(level - 1)
        for _ in range(prm.mu):
            mg_cycle_generic(b, level - 1, p, rc)
    b.add_prolonged(level, p, prm.tau if prm.damp_coarse else 1.0, u)
    for _ in range(prm.nu):
        z = b.smooth(level, b.residual(level, f, u))
        b.axpy_acc(prm.tau, z, u)


def mg_precondition(b, r):
    """multigrid.hpp:144-149"""
    z = b.zero_acc(b.finest_level())
    mg_cycle_generic(b, b.finest_level(), z, r)
    return z


def pcg_generic(b, f, tol: float, max_iter: int, precond, history: list):
    """multigrid.hpp:155-189"""
    L = b.finest_level()
    u = b.zero_acc(L)
    r = b.copy(f)

    def norm2(v):
        return math.sqrt(b.dot(L, v, b.accumulate(L, v)))

    r0 = norm2(r)
    history.clear()
    history.append(r0)
    if r0 == 0.0:
        return u
    z = precond(r)
    p = b.copy(z)
    rz = b.dot(L, r, z)
    for _ in range(1, max_iter + 1):
        Ap = b.apply_op(L, p)
        pAp = b.dot(L, Ap, p)
        if not pAp > 0.0:
            raise DefinitenessError("pcg: search direction with nonpositive energy")
        alpha = rz / pAp
        b.axpy_acc(alpha, p, u)
        b.axpy_dist(-alpha, Ap, r)
        rn = norm2(r)
        history.append(rn)
        if rn <= tol * r0:
            return u
        z = precond(r)
        rz_next = b.dot(L, r, z)
        b.xpay_acc(z, rz_next / rz, p)
        rz = rz_next
    raise DivergenceError("pcg: no convergence within the iteration limit")
