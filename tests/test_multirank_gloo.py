"""The multi-rank exchange protocol on CPU: world_size 2 over torch.distributed
(gloo, 127.0.0.1).  Each process takes its rank plan (csrc/common/
rank_plan.hpp -- the plan libpmg_cuda builds for its NCCL/hub exchanges),
forms its replica partial sums, exchanges them with its neighbours in plan
order, and folds the sources in ascending rank order.  The result must equal,
bitwise, the single-process fold of the reference (ParallelBackend::accumulate,
parallel.cpp:306-337); the scalar and coarse reductions follow the same
allgather / gather-to-0 + ascending-rank-sum protocol as the CUDA path."""
import ctypes as C
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1804_02539_b200 import Hierarchy
from paper_1804_02539_b200 import _native as N
from paper_1804_02539_b200.parallel import contiguous_partition


def plan(h, level, ranks, rank):
    v = N.PmghRankPlanView()
    assert N.host_lib().pmgh_rank_plan(h._h, level, ranks, rank, C.byref(v)) == 0
    n = v.n_iface
    arr = lambda p, k: np.ctypeslib.as_array(p, shape=(k,)).copy() if k else np.zeros(0, dtype=np.int32)  # noqa: E731
    rep_off = arr(v.rep_off, n + 1)
    comb_off = arr(v.comb_off, n + 1)
    nb_off = arr(v.nb_off, v.n_neighbors + 1)
    return {
        "iface_g": arr(v.iface_g, n), "rep_off": rep_off, "rep_slot": arr(v.rep_slot, int(rep_off[-1])),
        "comb_off": comb_off, "comb_src": arr(v.comb_src, int(comb_off[-1])),
        "nb_rank": arr(v.nb_rank, v.n_neighbors), "nb_off": nb_off, "nb_iface": arr(v.nb_iface, int(nb_off[-1])),
    }


def shares(h, level, seed):
    """A random distributed vector as per-patch lattice shares (all patches)."""
    rng = np.random.default_rng(seed)
    lat = rng.integers(-8, 9, size=(h.num_patches, h.lattice_size(level))).astype(np.float64) / 8.0
    lat[h.l2g(level) < 0] = 0.0
    return lat


def reference_fold(h, level, lat, ranks):
    """Per global dof: per-rank partials (ascending slot), summed in ascending rank order."""
    l2g = h.l2g(level)
    total = {}
    for r, (b, e) in enumerate(contiguous_partition(h.num_patches, ranks)):
        part = {}
        for k in range(b, e):
            for f in np.nonzero(l2g[k] >= 0)[0]:
                g = int(l2g[k, f])
                part[g] = part.get(g, 0.0) + lat[k, f]
        for g, v in part.items():
            total.setdefault(g, []).append(v)
    out = {}
    for g, vals in total.items():
        s = 0.0
        for v in vals:
            s += v
        out[g] = s
    return out


def worker(rank, world, port, dom, p, lv, n0, q):
    try:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
        h = Hierarchy(dom, p, lv, n0=n0)
        ok = []
        for level in range(h.num_levels):
            pl = plan(h, level, world, rank)
            lat_all = shares(h, level, 100 + level)
            b, e = contiguous_partition(h.num_patches, world)[rank]
            local = lat_all[b:e].reshape(-1)
            n = len(pl["iface_g"])
            tloc = np.array([_ordered_sum(local[pl["rep_slot"][pl["rep_off"][i]:pl["rep_off"][i + 1]]])
                             for i in range(n)])
            # neighbour exchange in plan order (NCCL grouped send/recv on the GPU)
            recv = np.zeros(len(pl["nb_iface"]))
            reqs = []
            for j, nb in enumerate(pl["nb_rank"]):
                lo, hi = pl["nb_off"][j], pl["nb_off"][j + 1]
                send = torch.from_numpy(tloc[pl["nb_iface"][lo:hi]].copy())
                rbuf = torch.zeros(hi - lo, dtype=torch.float64)
                reqs.append((dist.isend(send, int(nb)), dist.irecv(rbuf, int(nb)), lo, rbuf))
            for sreq, rreq, lo, rbuf in reqs:
                sreq.wait()
                rreq.wait()
                recv[lo:lo + len(rbuf)] = rbuf.numpy()
            t = np.zeros(n)
            for i in range(n):
                s = 0.0
                for q_ in range(pl["comb_off"][i], pl["comb_off"][i + 1]):
                    src = pl["comb_src"][q_]
                    s += tloc[i] if src < 0 else recv[src]
                t[i] = s
            ref = reference_fold(h, level, lat_all, world)
            ok.append(all(t[i] == ref[int(g)] for i, g in enumerate(pl["iface_g"])))
            # interface dofs are exactly the locally present dofs with >= 2 replicas overall
            off, _, _ = h.reps(level)
            counts = np.diff(off)
            present = np.zeros(h.num_dofs(level), dtype=bool)
            l2g_loc = h.l2g(level)[b:e]
            present[l2g_loc[l2g_loc >= 0]] = True
            ok.append(np.array_equal(np.sort(pl["iface_g"]), np.nonzero(present & (counts >= 2))[0]))
        # scalar reduction: allgather + ascending-rank sum, identical on every rank
        part = torch.tensor([float(rank) * 0.1 + 1.0 / 3.0], dtype=torch.float64)
        gathered = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(gathered, part)
        s = 0.0
        for g_ in gathered:
            s += float(g_[0])
        expect = 0.0
        for r in range(world):
            expect += float(r) * 0.1 + 1.0 / 3.0
        ok.append(s == expect)
        allres = [None] * world
        dist.all_gather_object(allres, s)
        ok.append(all(v == allres[0] for v in allres))
        q.put((rank, all(ok)))
        dist.destroy_process_group()
    except Exception as exc:  # noqa: BLE001
        q.put((rank, repr(exc)))


def _ordered_sum(v):
    s = 0.0
    for x in v:
        s += x
    return s


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("case", [("c2", 4, 2, 2), ("fichera", 2, 1, 1), ("c5", 3, 1, 2)])
def test_exchange_protocol_world2(case):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, 2, port, *case, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    res = dict(q.get(timeout=300) for _ in procs)
    for pr in procs:
        pr.join(timeout=60)
    assert res == {0: True, 1: True}, res
