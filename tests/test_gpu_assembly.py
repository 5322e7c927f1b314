"""Device stiffness assembly (assembly.cpp:127-248 restated
as a sum-factorized contraction, csrc/cuda/assembly.cu) against the host
assembly that the oracle uses.  The two differ only in summation order, so
the operators agree to 1e-13 relative and the PCG solve through the
device-assembled hierarchy matches the oracle as the host one does."""
import numpy as np
import pytest

import oracle
from paper_1804_02539_b200 import Hierarchy
from paper_1804_02539_b200.backend import GpuBackend

pytestmark = pytest.mark.gpu

CASES = [
    ("lshape", 2, 3, 1),
    ("two_squares_flipped_D", 3, 3, 1),
    ("c1", 2, 4, 2),
    ("c2", 4, 3, 2),
    ("c3", 5, 3, 2),
    ("c3", 8, 3, 2),
    ("fichera", 1, 3, 1),
    ("fichera", 2, 3, 1),
    ("c4", 3, 2, 2),
    ("c5", 3, 2, 2),
    ("c4", 4, 2, 1),
]


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


@pytest.mark.parametrize("dom,p,lv,n0", CASES, ids=[f"{c[0]}-p{c[1]}-L{c[2]}" for c in CASES])
def test_device_band_matches_host(dom, p, lv, n0):
    hh = Hierarchy(dom, p, lv, n0=n0)
    hd = Hierarchy(dom, p, lv, n0=n0, assembly="device")
    bh, bd = GpuBackend(hh), GpuBackend(hd)
    assert bd.assembly_seconds() > 0.0 and bh.assembly_seconds() == 0.0
    rng = np.random.default_rng(5)
    for level in range(hh.num_levels):
        u = rng.uniform(-1.0, 1.0, hh.num_dofs(level))
        yh = bh.gather_global(level, bh.apply_op(level, bh.to_accumulated(level, u)))
        yd = bd.gather_global(level, bd.apply_op(level, bd.to_accumulated(level, u)))
        assert rel(yd, yh) < 1e-13, level


@pytest.mark.parametrize("dom,p,lv,n0", [("c2", 4, 5, 2), ("c4", 3, 3, 2), ("fichera", 2, 4, 1)])
def test_pcg_on_device_assembled_hierarchy(dom, p, lv, n0):
    hh = Hierarchy(dom, p, lv, n0=n0)
    hd = Hierarchy(dom, p, lv, n0=n0, assembly="device")
    f = hh.rhs()
    assert np.array_equal(f, hd.rhs())
    u_ref, hist_ref, _, _ = oracle.Oracle(hh).pcg_solve(f)
    u, rep = GpuBackend(hd).pcg_solve(f)
    assert rep.iterations == len(hist_ref) - 1
    assert rel(u, u_ref) < 1e-10


@pytest.mark.parametrize("dom,p,lv,n0,env", [
    ("c2", 4, 5, 2, {}), ("c2", 4, 5, 2, {"PMG_SWEEP_MIN_EXT": "1"}),  # offset-major and line-major levels
    ("c2", 4, 4, 2, {"PMG_FULL_BAND": "1"}), ("c4", 3, 3, 2, {}), ("c3", 8, 3, 2, {}), ("fichera", 2, 3, 1, {}),
    ("c4", 3, 3, 2, {"PMG_SWEEP3D": "12"})])  # plane-major band of the 3D plane sweep
def test_band_download_feeds_the_oracle(dom, p, lv, n0, env, monkeypatch):
    """pmg_band_download: a device-assembled hierarchy hands its bands to the
    host (Hierarchy.adopt_device_bands); the oracle on those bands applies the
    host-assembled operator to 1e-13 on every level and its PCG matches the
    GPU's iteration count and solution."""
    for k, v in env.items():
        monkeypatch.setenv(k, v)
    hh = Hierarchy(dom, p, lv, n0=n0)
    hd = Hierarchy(dom, p, lv, n0=n0, assembly="device")
    bd = GpuBackend(hd)
    hd.adopt_device_bands(bd)
    od, oh = oracle.Oracle(hd), oracle.Oracle(hh)
    rng = np.random.default_rng(9)
    for level in range(hh.num_levels):
        u = rng.uniform(-1.0, 1.0, hh.num_dofs(level))
        assert rel(od.apply_op(level, u), oh.apply_op(level, u)) < 1e-13, level
    f = hd.rhs()
    u_ref, hist_ref, _, _ = od.pcg_solve(f)
    u, rep = bd.pcg_solve(f)
    assert rep.iterations == len(hist_ref) - 1
    assert rel(u, u_ref) < 1e-10


@pytest.mark.parametrize("dom,p,lv,n0,rhs", [
    ("c1", 2, 4, 2, "default"),          # sine_pi
    ("c2", 4, 4, 2, "default"),          # random nodes, perturbed 2D maps
    ("c3", 5, 3, 2, "one"),
    ("c4", 3, 3, 2, "default"),          # random nodes, jittered trilinear maps
    ("c5", 2, 2, 2, "default"),
    ("lshape", 2, 3, 1, "sine2d"),
    ("two_squares_flipped_D", 3, 3, 1, "sine2d"),
    ("fichera", 2, 3, 1, "sine3d"),
    ("fichera", 3, 2, 1, "one"),
])
def test_device_load_vector_matches_host(dom, p, lv, n0, rhs):
    """pmg_assemble_load (sum-factorized load vector on the device, a
    DistributedVector) against the host assemble_rhs restatement
    (assembly.cpp:299-365): every source kind, 2D and 3D, the seeded node
    values bit-identical (same counter-based generator), entries within 1e-13
    of the largest; a solve from the device-assembled vector has the oracle's
    iteration count and solution."""
    h = Hierarchy(dom, p, lv, n0=n0, rhs=rhs)
    b = GpuBackend(h)
    f_host = h.rhs()
    L = h.finest_level
    f_dev = b.assemble_load(rhs)
    got = b.gather_global(L, f_dev)
    assert np.abs(got - f_host).max() <= 1e-13 * np.abs(f_host).max()
    # Dirichlet slots of the distributed lattice vector are zero
    lat = f_dev.lattice().reshape(h.num_patches, -1)
    assert np.all(lat[h.l2g(L) < 0] == 0.0)
    # a hierarchy built without the host loop (rhs="zero") gives the same vector
    hz = Hierarchy(dom, p, lv, n0=n0, rhs="zero")
    assert not hz.rhs().any()
    bz = GpuBackend(hz)
    assert np.array_equal(bz.gather_global(L, bz.assemble_load(rhs)), got)
    u, rep = b.pcg_solve_device(f_dev)
    u_ref, hist_ref, _, _ = oracle.Oracle(h).pcg_solve(f_host)
    assert rep.iterations == len(hist_ref) - 1
    ug = b.gather_global(L, u)
    assert np.abs(ug - u_ref).max() <= 1e-10 * np.abs(u_ref).max()
