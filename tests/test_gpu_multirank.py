"""The multi-rank data path on one GPU: R contexts, each owning a contiguous
patch block, exchange interface sums, scalar reductions and the coarse
residual through the in-process hub (host-mediated device copies; no kernel
waits on another rank).  The same plans, packing and ordered folds run over
NCCL under torchrun.  Mirrors test_parallel.cpp:278-625."""
import numpy as np
import pytest

import oracle
from paper_1804_02539_b200 import Hierarchy
from paper_1804_02539_b200.parallel import local_dof_mask, parallel_pcg_solve, run_ranks

pytestmark = pytest.mark.gpu

CASES = [("c2", 4, 3, 2, "default"), ("fichera", 2, 2, 1, "sine3d"), ("c5", 3, 2, 2, "default"),
         ("c4", 3, 2, 2, "default")]


@pytest.fixture(scope="module", params=CASES, ids=[c[0] for c in CASES])
def hier(request):
    dom, p, lv, n0, rhs = request.param
    h = Hierarchy(dom, p, lv, n0=n0, rhs=rhs)
    return h, oracle.Oracle(h)


def rand(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


@pytest.mark.parametrize("R", [2, 4])
def test_operations_match_serial(hier, R):  # test_parallel.cpp:278-524
    h, o = hier
    L = h.finest_level
    g = rand(h.num_dofs(L), 7)
    u = rand(h.num_dofs(L), 8)
    g0 = rand(h.num_dofs(0), 9)
    ref_smooth = o.smooth(L, g)
    ref_coarse = o.coarse_solve(g0)
    ref_au = o.apply_op(L, u)

    def body(r, b):
        acc = b.gather_global(L, b.accumulate(L, b.to_distributed_owner(L, g)))
        sm = b.gather_global(L, b.smooth(L, b.to_distributed_owner(L, g)))
        au = b.apply_op(L, b.to_accumulated(L, u))
        au_loc = b.gather_global(L, au)
        cs = b.gather_global(0, b.coarse_solve(b.to_distributed_owner(0, g0)))
        dt = b.dot(L, b.to_distributed_owner(L, g), b.to_accumulated(L, u))
        return acc, sm, au_loc, cs, dt

    out = run_ranks(h, R, body)
    for r, (acc, sm, au_loc, cs, dt) in enumerate(out):
        m = local_dof_mask(h, L, r, R)
        m0 = local_dof_mask(h, 0, r, R)
        # accumulate reassembles the owner split exactly (test_parallel.cpp:278-376)
        assert np.array_equal(acc[m], g[m])
        assert np.abs(sm[m] - ref_smooth[m]).max() <= 1e-12 * np.abs(ref_smooth).max()
        assert np.abs(cs[m0] - ref_coarse[m0]).max() <= 1e-12 * np.abs(ref_coarse).max()
        assert dt == out[0][4]  # every rank holds the same reduced bits
        assert abs(dt - g @ u) <= 1e-13 * np.abs(g * u).sum()
    # apply_op shares sum to the serial operator
    total = sum(o_[2] for o_ in out)
    assert np.abs(total - ref_au).max() <= 1e-13 * (1 + np.abs(ref_au).max())


@pytest.mark.parametrize("R", [2, 4])
def test_parallel_solve_tracks_serial(hier, R):  # test_parallel.cpp:581-625
    h, o = hier
    f = h.rhs()
    u_ser, hist_ser, _, _ = o.pcg_solve(f)
    u_par, hist_par, _, _ = o.pcg_solve(f, ranks=R)
    u, rep, nbytes = parallel_pcg_solve(h, R, f)
    assert nbytes > 0
    assert rep.iterations == len(hist_ser) - 1 == len(hist_par) - 1
    scale = np.abs(u_ser).max()
    assert np.abs(u - u_ser).max() <= 1e-10 * scale
    hist = np.array(rep.residual_history)
    k = min(5, len(hist))
    assert np.all(np.abs(hist[:k] - hist_ser[:k]) <= 1e-10 * hist_ser[:k])
    # same partition, same exchange order: a rerun reproduces every bit
    _, rep2, _ = parallel_pcg_solve(h, R, f)
    assert rep2.residual_history == rep.residual_history


@pytest.mark.parametrize("R", [2, 4])
def test_concurrent_line_sweeps(R, monkeypatch):
    """R contexts solve at once on one GPU with the 2D line sweep on every
    level (PMG_SWEEP_MIN_EXT=1): each rank's sweep grid is sized to fill the
    GPU alone, so the grids compete for SMs.  A sweep CTA waits for the carry
    of the segment above it; segments are handed out in CTA start order, so the
    wait never depends on co-residency.  The solve must finish and match the
    serial iteration count and solution."""
    monkeypatch.setenv("PMG_SWEEP_MIN_EXT", "1")
    h = Hierarchy("c2", 4, 5, n0=2)
    o = oracle.Oracle(h)
    f = h.rhs()
    u_ref, hist_ref, _, _ = o.pcg_solve(f)
    u, rep, _ = parallel_pcg_solve(h, R, f)
    assert rep.iterations == len(hist_ref) - 1
    assert np.abs(u - u_ref).max() <= 1e-10 * np.abs(u_ref).max()


@pytest.mark.parametrize("dom,p,lv,n0,rhs", [("c3", 4, 4, 2, "default"), ("unit_grid(2,2,2)", 2, 3, 2, "sine3d")])
@pytest.mark.parametrize("R", [2, 4])
def test_matrix_free_and_device_load_on_ranks(dom, p, lv, n0, rhs, R):
    """Round-2 paths on R ranks: the Kronecker operator (PMG_BAND_KRONECKER)
    applies each rank's patches with that rank's geometry factors, and
    pmg_assemble_load assembles each rank's share of the load vector (the
    seeded node values indexed by the global patch number).  The shares sum to
    the host vector; the solve has the serial iteration count and solution."""
    h = Hierarchy(dom, p, lv, n0=n0, rhs=rhs, operator="kronecker")
    o = oracle.Oracle(h)
    L = h.finest_level
    f = h.rhs()
    u_ref, hist_ref, _, _ = o.pcg_solve(f)
    x = rand(h.num_dofs(L), 3)
    ref_ax = o.apply_op(L, x)

    def body(r, b):
        fd = b.assemble_load(rhs)
        share = b.gather_global(L, fd)
        ax = b.gather_global(L, b.apply_op(L, b.to_accumulated(L, x)))
        u, rep = b.pcg_solve_device(fd)
        return share, ax, b.gather_global(L, u), rep.iterations

    out = run_ranks(h, R, body)
    assert np.abs(sum(o_[0] for o_ in out) - f).max() <= 1e-13 * np.abs(f).max()
    assert np.abs(sum(o_[1] for o_ in out) - ref_ax).max() <= 1e-13 * np.abs(ref_ax).max()
    for r, (_, _, u, its) in enumerate(out):
        m = local_dof_mask(h, L, r, R)
        assert its == len(hist_ref) - 1
        assert np.abs(u[m] - u_ref[m]).max() <= 1e-10 * np.abs(u_ref).max()
