"""CUDA path vs the CPU oracle at BASELINE.json's FULL sizes: c2 (1,071,225
dofs), c3 at p = 2, 3, 4, 6, 8 (128^2 elements per patch), c4 (2,317,259 dofs)
and c5 (9,269,435 dofs).

The oracle runs the reference's own rank-parallel semantics
(parallel_pcg_solve over R = min(host threads, patches) in-process ranks,
parallel.cpp:497-518) on every host thread, next to the GPU solve of the same
hierarchy.  c2 and c3 are assembled on the host (the oracle's usual input).
c4 and c5 are assembled on the device -- stiffness and load vector -- and
the bands and the load vector are downloaded to the host
(Hierarchy.adopt_device_bands, pmg_assemble_load), so both sides apply the
same operator to the same right-hand side; device vs host assembly is checked
separately (test_gpu_assembly.py, and with PMG_TEST_FULL=1
test_device_assembly_matches_host_assembly below at full c4).  The default
selection runs c2, c3 at p = 2 and 8, c4 and c5, the 3D ones against the
first six oracle iterations (the driver's 20-minute limit; the oracle needs
4-12 s per c5 iteration on this pool's hosts); PMG_TEST_FULL=1 adds
p = 3, 4, 6 and runs every oracle solve to convergence -- that run is the
committed record.

Asserted (north_star, BASELINE.json; reference window multigrid.hpp:155-189,
multigrid.cpp:72-89):
  * identical PCG iteration counts;
  * the solution within 1e-10 relative (max norm);
  * every residual norm ||r_k|| >= 1e-4 ||r_0|| within 1e-10 RELATIVE to
    ||r_k|| -- the reference's own serial-vs-parallel check compares its first
    iterations at 1e-10 (test_parallel.cpp:581-625) -- or, where the coarse
    matrix is so ill-conditioned that two exact coarse solvers inside the
    oracle (LLT substitution vs explicit inverse) already differ by more
    (c3 at p = 8, kappa(A_0) = 3e7), within twice that measured spread;
  * the tail (||r_k|| < 1e-4 ||r_0||) within 1e-10 ||r_k|| + floor ||r_0||,
    floor = max(1e-12, 1e-3 kappa(A_0) eps): two fp64 implementations that
    sum in different orders keep an O(eps ||r_0||) gap in the recursively
    updated residual;
  * the finest-level operators (apply_op, residual, smooth, restriction,
    prolongation, V-cycle) against the oracle at 1e-13 / 1e-12 / 1e-11, and
    the smoother with every fast-diagonalization column panel forced
    (PMG_FD_NTC = 3, 5, 9, 11; the bench's c2 finest level selects 9).

The measured deviations are written to $PMG_PARITY_RECORD (default
gpurun_out/parity_fullsize.json), one JSON object per config; the committed
copy is profiles/parity_fullsize_r02.json."""
import json
import os
import time
from pathlib import Path

import numpy as np
import pytest

import oracle
from paper_1804_02539_b200.backend import GpuBackend
from paper_1804_02539_b200.hierarchy import CONFIGS, Hierarchy

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ROOT = Path(__file__).resolve().parents[1]
RECORD = Path(os.environ.get("PMG_PARITY_RECORD", ROOT / "gpurun_out" / "parity_fullsize.json"))
from tests.helpers import FULL_MATRIX  # noqa: E402

# default: every BASELINE family; PMG_TEST_FULL=1 adds the two remaining c3 degrees
FULL = (["c2", "c3p2", "c3p3", "c3p4", "c3p6", "c3p8", "c4", "c5"] if FULL_MATRIX
        else ["c2", "c3p2", "c3p8", "c4", "c5"])
HEAD_ITS = 6
DEVICE = ("c4", "c5")  # stiffness and load vector assembled on the device (host: 32 s + 13 s at c4, minutes at c5)


def record(name, **kv):
    RECORD.parent.mkdir(parents=True, exist_ok=True)
    data = json.loads(RECORD.read_text()) if RECORD.exists() else {}
    data.setdefault(name, {}).update(kv)
    RECORD.write_text(json.dumps(data, indent=1, sort_keys=True))


def rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def rand(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


@pytest.fixture(scope="module", params=FULL)
def full(request):
    name = request.param
    dom, p, n0, lv = CONFIGS[name]
    assembly = "device" if name in DEVICE else "host"
    t0 = time.perf_counter()
    h = Hierarchy(dom, p, lv, n0=n0, assembly=assembly, rhs="zero" if assembly == "device" else "default")
    t_setup = time.perf_counter() - t0
    b = GpuBackend(h)
    t_dl = h.adopt_device_bands(b) if assembly == "device" else 0.0
    o = oracle.Oracle(h)
    record(name, dofs=h.num_dofs(h.finest_level), assembly=h.assembly, host_setup_s=t_setup, band_download_s=t_dl)
    # the load vector both solvers get: the host's, or (device-assembled configs) the device's, downloaded
    h.load_vector = (b.gather_global(h.finest_level, b.assemble_load("default")) if assembly == "device"
                     else h.rhs())
    yield name, h, b, o
    b.close()
    del o


def test_finest_operators(full):
    name, h, b, o = full
    L = h.finest_level
    n = h.num_dofs(L)
    u, f = rand(n, 1), rand(n, 2)
    dev = {}
    dev["apply_op"] = rel(b.gather_global(L, b.apply_op(L, b.to_accumulated(L, u))), o.apply_op(L, u))
    dev["residual"] = rel(b.gather_global(L, b.residual(L, b.to_distributed_owner(L, f), b.to_accumulated(L, u))),
                          o.residual(L, f, u))
    ref_smooth = o.smooth(L, f)
    dev["smooth"] = rel(b.gather_global(L, b.smooth(L, b.to_distributed_owner(L, f))), ref_smooth)
    dev["restrict"] = rel(b.gather_global(L - 1, b.restrict_residual(L, b.to_distributed_owner(L, f))),
                          o.restrict(L, f))
    c = rand(h.num_dofs(L - 1), 3)
    ug = b.to_accumulated(L, u)
    b.add_prolonged(L, b.to_accumulated(L - 1, c), 0.7, ug)
    dev["add_prolonged"] = rel(b.gather_global(L, ug), o.add_prolonged(L, c, 0.7, u))
    # the oracle's V-cycle is serial (40 s at c5): at c5 it is compared only with PMG_TEST_FULL=1 -- the PCG
    # parity below runs it 24 times through the rank-parallel oracle
    if name != "c5" or FULL_MATRIX:
        dev["precondition"] = rel(b.gather_global(L, b.precondition(b.to_distributed_owner(L, f))), o.precondition(f))
    record(name, operator_rel_dev=dev)
    assert dev["apply_op"] < 1e-13 and dev["residual"] < 1e-13, dev
    assert dev["restrict"] < 1e-13 and dev["add_prolonged"] < 1e-13, dev
    assert dev["smooth"] < 1e-12, dev
    assert dev.get("precondition", 0.0) < 1e-11, dev
    if name == "c2" or (FULL_MATRIX and name == "c4"):
        # every fast-diagonalization column panel on the finest level
        panels = {}
        for ntc in ("3", "5", "9", "11"):
            os.environ["PMG_FD_NTC"] = ntc
            try:
                bf = GpuBackend(h)
                panels[ntc] = rel(bf.gather_global(L, bf.smooth(L, bf.to_distributed_owner(L, f))), ref_smooth)
                bf.close()
            finally:
                del os.environ["PMG_FD_NTC"]
        record(name, smooth_rel_dev_forced_panels=panels)
        assert all(v < 1e-12 for v in panels.values()), panels


def test_pcg_matches_oracle(full):
    name, h, b, o = full
    L = h.finest_level
    f = h.load_vector
    ranks = max(1, min(os.cpu_count() or 1, h.num_patches))
    # The oracle needs 4-12 s per iteration at c5 on this pool's hosts.  Under the driver's 20-minute limit
    # the default selection therefore runs it for the first HEAD_ITS iterations of the 3D configs and
    # compares those residual norms (the reference's own parallel-vs-serial test compares five,
    # test_parallel.cpp:581-625); PMG_TEST_FULL=1 runs it to convergence (iteration count, solution, whole
    # history: profiles/parity_fullsize_r02.json holds that run).
    head_only = name in DEVICE and not FULL_MATRIX
    if head_only:
        u_ref, hist_ref, t_ref, _ = o.pcg_solve(f, max_iter=HEAD_ITS, allow_cap=True, ranks=ranks)
    else:
        u_ref, hist_ref, t_ref, _ = o.pcg_solve(f, ranks=ranks)
    t0 = time.perf_counter()
    u, rep = b.pcg_solve(f)
    t_gpu = time.perf_counter() - t0
    hist = np.array(rep.residual_history)
    if head_only:
        k = len(hist_ref)
        assert k == HEAD_ITS + 1 and rep.iterations >= HEAD_ITS
        relk = np.abs(hist[:k] - hist_ref) / hist_ref
        record(name, head_only_iterations=HEAD_ITS, head_only_max_rel_dev=float(relk.max()),
               head_only_iterations_gpu=rep.iterations)
        assert np.all(relk <= 1e-10), relk
        assert hist[-1] <= 1e-8 * hist[0] and rep.iterations < 60
        return
    k = min(len(hist), len(hist_ref))
    d = np.abs(hist[:k] - hist_ref[:k])
    relk = d / hist_ref[:k]
    head = hist_ref[:k] >= 1e-4 * hist_ref[0]
    kappa = float(np.linalg.cond(h.coarse_matrix()))
    floor = max(1e-12, 1e-3 * kappa * np.finfo(float).eps)
    u_dev = rel(u, u_ref)
    # conditioning limit of the coarse solve: where kappa(A_0) eps is not
    # negligible, two EXACT coarse solvers (the oracle's LLT substitution and
    # the explicit inverse the GPU applies, both in the oracle) already differ
    # by more than 1e-10 in the head of the residual history (c3 at p = 8:
    # kappa(A_0) = 3e7).  The head bound is then twice that measured spread.
    coarse_limit = 0.0
    if kappa * np.finfo(float).eps > 1e-11:
        o.set_coarse_mode(1)
        try:
            _, hist_inv, _, _ = o.pcg_solve(f, ranks=ranks)
        finally:
            o.set_coarse_mode(0)
        kk = min(len(hist_inv), k)
        dd = np.abs(hist_inv[:kk] - hist_ref[:kk]) / hist_ref[:kk]
        coarse_limit = float(dd[head[:kk]].max())
    head_bound = max(1e-10, 2.0 * coarse_limit)
    record(name, iterations_gpu=rep.iterations, iterations_oracle=len(hist_ref) - 1, oracle_ranks=ranks,
           oracle_solve_s=t_ref, gpu_solve_s_incl_copies=t_gpu, u_rel_dev=u_dev,
           max_rel_dev_head=float(relk[head].max()), head_iterations=int(head.sum()),
           max_rel_dev_all=float(relk.max()), max_abs_dev_over_r0=float(d.max() / hist_ref[0]),
           rel_dev_per_iteration=[float(x) for x in relk], final_rel_residual=float(hist_ref[-1] / hist_ref[0]),
           kappa_A0=kappa, floor=floor, oracle_llt_vs_inverse_head_rel_dev=coarse_limit, head_bound=head_bound)
    assert rep.iterations == len(hist_ref) - 1
    assert u_dev < 1e-10
    assert np.all(relk[head] <= head_bound), relk
    assert np.all(d <= 1e-10 * hist_ref[:k] + floor * hist_ref[0]), relk


@pytest.mark.skipif(not FULL_MATRIX, reason="PMG_TEST_FULL=1: 32 s of host assembly; desk sizes in test_gpu_assembly.py")
def test_device_assembly_matches_host_assembly():
    """Full c4: the operator assembled on the device against the oracle on the
    host assembly of the reference (assembly.cpp:127-248), every level."""
    dom, p, n0, lv = CONFIGS["c4"]
    hh = Hierarchy(dom, p, lv, n0=n0, assembly="host")
    hd = Hierarchy(dom, p, lv, n0=n0, assembly="device")
    bd = GpuBackend(hd)
    oh = oracle.Oracle(hh)
    worst = {}
    for level in range(1, hh.num_levels):
        u = rand(hh.num_dofs(level), 40 + level)
        worst[level] = rel(bd.gather_global(level, bd.apply_op(level, bd.to_accumulated(level, u))),
                           oh.apply_op(level, u))
    bd.close()
    record("c4", device_vs_host_assembly_apply_rel_dev=worst)
    assert max(worst.values()) < 1e-13, worst
