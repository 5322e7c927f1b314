"""Matrix-free Kronecker operator (PMG_BAND_KRONECKER)
against the oracle, which applies the host-assembled band exactly as the
reference does (assembly.cpp:12-18,265-280).  On axis-aligned affine patches
the assembled stiffness is the Kronecker sum of the univariate matrices
(test_assembly.cpp:112-146), so the two agree to rounding: operators within
1e-13, identical PCG iteration counts, u within 1e-10 (north_star)."""
import numpy as np
import pytest

from paper_1804_02539_b200 import Hierarchy
from paper_1804_02539_b200.backend import GpuBackend
from paper_1804_02539_b200.errors import ConfigError

import oracle

pytestmark = pytest.mark.gpu

CASES = [
    ("c1", 2, 5, 2, "default"),
    ("c3", 1, 5, 2, "default"),
    ("c3", 3, 5, 2, "default"),
    ("c3", 4, 4, 2, "default"),
    ("c3", 6, 5, 2, "default"),
    ("c3", 8, 5, 2, "default"),
    ("lshape", 2, 4, 1, "one"),
    ("two_squares_flipped_D", 3, 3, 1, "sine2d"),  # a patch map with h < 0
    ("unit_grid(3,2)", 5, 3, 2, "sine2d"),
    ("fichera", 2, 3, 1, "sine3d"),
    ("fichera", 3, 2, 1, "sine3d"),
    ("unit_grid(2,2,2)", 3, 3, 2, "sine3d"),
    ("unit_grid(2,1,2)", 1, 3, 2, "sine3d"),
]
IDS = [f"{c[0]}-p{c[1]}-L{c[2]}" for c in CASES]


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def rand(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


@pytest.mark.parametrize("dom,p,lv,n0,rhs", CASES, ids=IDS)
def test_kronecker_operator_matches_oracle(dom, p, lv, n0, rhs):
    h = Hierarchy(dom, p, lv, n0=n0, rhs=rhs, operator="kronecker")
    b, o = GpuBackend(h), oracle.Oracle(h)
    for level in range(h.num_levels):
        n = h.num_dofs(level)
        u, f = rand(n, 1 + level), rand(n, 100 + level)
        got = b.gather_global(level, b.apply_op(level, b.to_accumulated(level, u)))
        assert rel(got, o.apply_op(level, u)) < 1e-13, level
        got = b.gather_global(level, b.residual(level, b.to_distributed_owner(level, f), b.to_accumulated(level, u)))
        assert rel(got, o.residual(level, f, u)) < 1e-13, level
    L = h.finest_level
    fz = rand(h.num_dofs(L), 3)
    z = b.gather_global(L, b.precondition(b.to_distributed_owner(L, fz)))
    assert rel(z, o.precondition(fz)) < 1e-11
    f = h.rhs()
    u_ref, hist_ref, _, _ = o.pcg_solve(f)
    u, rep = b.pcg_solve(f)
    assert rep.iterations == len(hist_ref) - 1
    assert rel(u, u_ref) < 1e-10
    # residual norms: the bound of test_gpu_parity.py::test_pcg_matches_oracle
    # (1e-10 relative plus the fp64 floor of the recursively updated residual)
    from tests.test_gpu_parity import history_floor
    hist = np.array(rep.residual_history)
    floor = history_floor(h, o, f, hist_ref)
    assert np.all(np.abs(hist - hist_ref) <= 1e-10 * hist_ref + floor * hist_ref[0])
    # bitwise reruns (deterministic dot partials)
    u2, rep2 = b.pcg_solve(f)
    assert np.array_equal(u, u2) and rep2.residual_history == rep.residual_history


@pytest.mark.parametrize("dom,p,lv,n0", [("c3", 8, 5, 2), ("unit_grid(2,2,2)", 3, 3, 2)])
def test_kronecker_matches_band_backend(dom, p, lv, n0):
    """Same hierarchy through the assembled half band and matrix-free."""
    hb = Hierarchy(dom, p, lv, n0=n0)
    hk = Hierarchy(dom, p, lv, n0=n0, operator="kronecker")
    bb, bk = GpuBackend(hb), GpuBackend(hk)
    L = hb.finest_level
    u = rand(hb.num_dofs(L), 5)
    yb = bb.gather_global(L, bb.apply_op(L, bb.to_accumulated(L, u)))
    yk = bk.gather_global(L, bk.apply_op(L, bk.to_accumulated(L, u)))
    assert rel(yk, yb) < 1e-13
    ub, rb = bb.pcg_solve(hb.rhs())
    uk, rk = bk.pcg_solve(hk.rhs())
    assert rb.iterations == rk.iterations
    assert rel(uk, ub) < 1e-10


@pytest.mark.parametrize("dom,p,lv,n0", [("c2", 4, 3, 2), ("c4", 3, 2, 2), ("c5", 2, 2, 2)])
def test_kronecker_rejects_other_geometry(dom, p, lv, n0):
    """Perturbed or trilinear-jittered patch maps are not a Kronecker
    sum: context creation is a ConfigError, never a silently wrong operator."""
    h = Hierarchy(dom, p, lv, n0=n0, operator="kronecker")
    with pytest.raises(ConfigError):
        GpuBackend(h)
