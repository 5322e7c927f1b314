"""Multi-rank solve path: patches partitioned across GPUs.

Restates the reference's rank-parallel layer (parallel.hpp:133-341,
parallel.cpp:181-518) on top of the CUDA contexts:

  contiguous_partition   patch blocks per rank (parallel.cpp:181-198)
  run_ranks              R ranks as threads of this process over an
                         in-process hub (InProcHub + run_ranks,
                         parallel.cpp:118-179); exchanges are host-mediated
                         device copies, so it runs on a single GPU too
  parallel_pcg_solve     the hub-driven solve (parallel.cpp:497-518)
  RankBackend            one process per GPU under torchrun, NCCL transport
                         (the unique id travels over torch.distributed)
"""
from __future__ import annotations

import ctypes as C
import threading

import numpy as np

from . import _native as N
from .backend import GpuBackend, SolveReport
from .errors import ConfigError, raise_for
from .hierarchy import Hierarchy

MAX_RANKS = 64  # kMaxRanks, parallel.hpp:24


def contiguous_partition(num_patches: int, ranks: int):
    """[(patch_begin, patch_end)] per rank (parallel.cpp:181-198)."""
    if ranks < 1:
        raise ConfigError("partition: need at least one rank")
    if ranks > MAX_RANKS:
        raise ConfigError("partition: rank cap exceeded")
    if ranks > num_patches:
        raise ConfigError("partition: more ranks than patches")
    return [(num_patches * r // ranks, num_patches * (r + 1) // ranks) for r in range(ranks)]


def comm_desc(rank: int, size: int, num_patches: int, transport: int, nccl_id: bytes | None = None,
              hub=None) -> N.PmgCommDesc:
    b, e = contiguous_partition(num_patches, size)[rank]
    d = N.PmgCommDesc()
    d.rank, d.size, d.patch_begin, d.patch_end, d.transport = rank, size, b, e, transport
    if nccl_id is not None:
        C.memmove(d.nccl_id, nccl_id, 128)
    d.hub = hub
    return d


class Hub:
    def __init__(self, ranks: int):
        self._lib = N.cuda_lib()
        h = C.c_void_p()
        raise_for(self._lib.pmg_hub_create(ranks, C.byref(h)), self._lib.pmg_last_error(None).decode())
        self.handle = h
        self.ranks = ranks

    def poison(self, reason: str):
        self._lib.pmg_hub_poison(self.handle, reason.encode())

    def __del__(self):
        try:
            self._lib.pmg_hub_destroy(self.handle)
        except Exception:
            pass


def local_dof_mask(h: Hierarchy, level: int, rank: int, size: int) -> np.ndarray:
    b, e = contiguous_partition(h.num_patches, size)[rank]
    mask = np.zeros(h.num_dofs(level), dtype=bool)
    l2g = h.l2g(level)[b:e]
    mask[l2g[l2g >= 0]] = True
    return mask


def run_ranks(h: Hierarchy, ranks: int, fn, device: int = 0):
    """fn(rank, backend) on one thread per rank; the first failure poisons the
    hub, every thread stops, and the failure is re-raised (run_ranks,
    parallel.cpp:153-179).  Returns the per-rank results."""
    hub = Hub(ranks)
    # contexts are created before the threads start (creation is collective-free)
    backends = [GpuBackend(h, device=device, comm=comm_desc(r, ranks, h.num_patches, N.PMG_TRANSPORT_HUB,
                                                            hub=hub.handle)) for r in range(ranks)]
    results = [None] * ranks
    errors = [None] * ranks
    first = []
    lock = threading.Lock()

    def body(r):
        try:
            results[r] = fn(r, backends[r])
        except BaseException as e:  # noqa: BLE001
            errors[r] = e
            with lock:
                if not first:
                    first.append(r)
            hub.poison("peer rank failed")

    threads = [threading.Thread(target=body, args=(r,)) for r in range(ranks)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    if first:
        raise errors[first[0]]
    for b in backends:
        b.close()
    return results


def parallel_pcg_solve(h: Hierarchy, ranks: int, f: np.ndarray, tol: float = 1e-8, max_iter: int = 500,
                       device: int = 0):
    """parallel_pcg_solve (parallel.cpp:497-518) over the in-process hub: every
    rank owner-masks the load vector (to_distributed_owner), runs the PCG on its
    patches, and the accumulated solution is gathered.  Returns
    (u, SolveReport of rank 0, total bytes pushed between ranks)."""
    L = h.finest_level

    def rank_solve(r, b: GpuBackend):
        fd = b.to_distributed_owner(L, f)
        u, rep = b.pcg_solve_device(fd, tol=tol, max_iter=max_iter)
        return b.gather_global(L, u), rep, b.comm_bytes()

    out = run_ranks(h, ranks, rank_solve, device=device)
    u = np.zeros(h.num_dofs(L))
    for r, (ur, _, _) in enumerate(out):
        mask = local_dof_mask(h, L, r, ranks)
        u[mask] = ur[mask]
    return u, out[0][1], sum(o[2] for o in out)


class RankBackend(GpuBackend):
    """One rank of a torchrun job (one process per GPU): NCCL over NVLink."""

    def __init__(self, h: Hierarchy, rank: int, world: int, local_rank: int):
        import torch.distributed as dist
        lib = N.cuda_lib()
        uid = (C.c_ubyte * 128)()
        if rank == 0:
            raise_for(lib.pmg_nccl_unique_id(C.byref(uid)), lib.pmg_last_error(None).decode())
        box = [bytes(uid)]
        dist.broadcast_object_list(box, src=0)
        super().__init__(h, device=local_rank,
                         comm=comm_desc(rank, world, h.num_patches, N.PMG_TRANSPORT_NCCL, nccl_id=box[0]))
        self._mask = local_dof_mask(h, h.finest_level, rank, world)

    def pcg_solve(self, f_global: np.ndarray, tol: float = 1e-8, max_iter: int = 500):
        """Host load vector in, this rank's share of the accumulated solution
        out (entries of dofs on other ranks are 0)."""
        L = self.h.finest_level
        fd = self.to_distributed_owner(L, f_global)
        u, rep = self.pcg_solve_device(fd, tol=tol, max_iter=max_iter)
        out = self.gather_global(L, u)
        out[~self._mask] = 0.0
        return out, rep


__all__ = ["contiguous_partition", "comm_desc", "Hub", "run_ranks", "parallel_pcg_solve", "RankBackend",
           "local_dof_mask", "SolveReport"]
