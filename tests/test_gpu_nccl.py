"""The NCCL transport on the GPU at world size 1 (one process, one GPU).

An NCCL job creates its rank transport at any world size, so a world-1
context runs every collective of the multi-GPU path through NCCL: the
grouped send/recv interface exchange (empty at one rank), the ncclAllGather
of the dot and norm partials with the ascending-rank fold, and the coarse
gather to rank 0 plus ncclBroadcast -- all captured into the PCG graphs.
The solve must agree with the single-GPU context (which issues no
collective) and with the oracle.  Reference: parallel.cpp:21-35 (ordered
all-reduce), :306-337 (accumulate), :411-422 (coarse solve)."""
import ctypes as C

import numpy as np
import pytest

import oracle
from paper_1804_02539_b200 import Hierarchy
from paper_1804_02539_b200 import _native as N
from paper_1804_02539_b200.backend import GpuBackend
from paper_1804_02539_b200.parallel import comm_desc

pytestmark = pytest.mark.gpu


def nccl_backend(h):
    lib = N.cuda_lib()
    uid = (C.c_ubyte * 128)()
    assert lib.pmg_nccl_unique_id(C.byref(uid)) == 0, lib.pmg_last_error(None)
    return GpuBackend(h, comm=comm_desc(0, 1, h.num_patches, N.PMG_TRANSPORT_NCCL, nccl_id=bytes(uid)))


def collectives(b):
    n = C.c_int64()
    assert N.cuda_lib().pmg_ctx_info(b._ctx, 6, C.byref(n)) == 0
    return n.value


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("dom,p,lv,n0", [("c2", 4, 4, 2), ("c4", 3, 3, 2), ("fichera", 2, 3, 1)])
def test_nccl_world1_solve(dom, p, lv, n0):
    h = Hierarchy(dom, p, lv, n0=n0)
    f = h.rhs()
    bn = nccl_backend(h)
    before = collectives(bn)
    u, rep = bn.pcg_solve(f)
    assert collectives(bn) > before  # the solve went through the transport
    u1, rep1 = GpuBackend(h).pcg_solve(f)
    u_ref, hist_ref, _, _ = oracle.Oracle(h).pcg_solve(f)
    assert rep.iterations == rep1.iterations == len(hist_ref) - 1
    assert rel(u, u1) < 1e-12 and rel(u, u_ref) < 1e-10
    # graph replay of the captured NCCL collectives reproduces every bit
    u2, rep2 = bn.pcg_solve(f)
    assert np.array_equal(u2, u)
    assert np.array_equal(np.array(rep2.residual_history), np.array(rep.residual_history))


def test_nccl_world1_operations():
    h = Hierarchy("c4", 3, 3, n0=2)
    bn, b1 = nccl_backend(h), GpuBackend(h)
    L = h.finest_level
    rng = np.random.default_rng(3)
    g = rng.uniform(-1, 1, h.num_dofs(L))
    g0 = rng.uniform(-1, 1, h.num_dofs(0))
    for b in (bn, b1):
        assert np.array_equal(b.gather_global(L, b.accumulate(L, b.to_distributed_owner(L, g))), g)
    d_n = bn.dot(L, bn.to_distributed_owner(L, g), bn.to_accumulated(L, g))
    d_1 = b1.dot(L, b1.to_distributed_owner(L, g), b1.to_accumulated(L, g))
    assert d_n == d_1  # a one-rank ordered fold is the identity
    cs_n = bn.gather_global(0, bn.coarse_solve(bn.to_distributed_owner(0, g0)))
    cs_1 = b1.gather_global(0, b1.coarse_solve(b1.to_distributed_owner(0, g0)))
    assert np.array_equal(cs_n, cs_1)
    sm_n = bn.gather_global(L, bn.smooth(L, bn.to_distributed_owner(L, g)))
    sm_1 = b1.gather_global(L, b1.smooth(L, b1.to_distributed_owner(L, g)))
    assert rel(sm_n, sm_1) < 1e-13
