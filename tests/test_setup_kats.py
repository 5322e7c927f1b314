"""Known-answer tests of the host setup library, ported from the reference's
test suite (the reference cannot be built here: Eigen3 is absent).  Each test
names the reference test it restates.  CPU only."""
import ctypes as C
import math

import numpy as np
import pytest
import scipy.linalg as sla

from paper_1804_02539_b200 import ConfigError, DecompositionError, Hierarchy
from paper_1804_02539_b200 import _native as N
from tests.helpers import band_offsets, eval_basis, gauss_legendre, global_matrix, gram, two_scale


# ---------------------------------------------------------------- test_spline.cpp
def test_gauss_legendre_rules():  # test_spline.cpp:29-59
    assert gauss_legendre(0)[0] == N.PMG_ERR_DOMAIN
    assert gauss_legendre(65)[0] == N.PMG_ERR_DOMAIN
    _, n1, w1 = gauss_legendre(1)
    assert n1[0] == pytest.approx(0.5) and w1[0] == pytest.approx(1.0)
    _, n2, _ = gauss_legendre(2)
    assert n2[0] == pytest.approx(0.5 - 0.5 / math.sqrt(3)) and n2[1] == pytest.approx(0.5 + 0.5 / math.sqrt(3))
    for q in range(1, 13):
        _, x, w = gauss_legendre(q)
        assert abs(w.sum() - 1.0) < 1e-14
        for k in range(2 * q):
            assert abs((w * x ** k).sum() - 1.0 / (k + 1)) < 1e-13
        assert np.all(np.diff(x) > 0) and x[0] > 0 and x[-1] < 1


def test_banded_cholesky():  # test_spline.cpp:61-88
    lib = N.host_lib()
    band = np.zeros((4, 2))
    band[:, 0] = 4.0
    band[1:, 1] = 1.0
    rhs = np.array([1.0, -2.0, 3.0, 0.5])
    x = np.zeros(4)
    assert lib.pmgh_banded_cholesky_solve(4, 1, band.ctypes.data_as(N._dp), rhs.ctypes.data_as(N._dp),
                                          x.ctypes.data_as(N._dp)) == 0
    dense = np.diag([4.0] * 4) + np.diag([1.0] * 3, 1) + np.diag([1.0] * 3, -1)
    assert np.abs(dense @ x - rhs).max() < 1e-13
    bad = np.array([[1.0, 0.0], [1.0, 2.0]])  # [[1,2],[2,1]] indefinite
    assert lib.pmgh_banded_cholesky_solve(2, 1, bad.ctypes.data_as(N._dp), rhs.ctypes.data_as(N._dp),
                                          x.ctypes.data_as(N._dp)) == N.PMG_ERR_DEFINITENESS


def test_basis_frozen_values():  # test_spline.cpp:112-140
    rc, f, v = eval_basis(1, 2, 0.25)
    assert f == 0 and v[0] == pytest.approx(0.5) and v[1] == pytest.approx(0.5)
    _, f, v = eval_basis(2, 1, 0.5)
    assert f == 0 and np.allclose(v, [0.25, 0.5, 0.25])
    _, f, v = eval_basis(2, 1, 0.0)
    assert v[0] == pytest.approx(1.0) and abs(v[1]) < 1e-15
    _, f, v = eval_basis(2, 1, 1.0)
    assert f == 0 and v[2] == pytest.approx(1.0)
    _, _, d = eval_basis(1, 2, 0.25, deriv=1)
    assert d[0] == pytest.approx(-2.0) and d[1] == pytest.approx(2.0)
    assert eval_basis(1, 2, -0.1)[0] == N.PMG_ERR_DOMAIN
    assert eval_basis(1, 2, 1.1)[0] == N.PMG_ERR_DOMAIN


def test_basis_partition_of_unity_and_marsden():  # test_spline.cpp:142-184
    rng = np.random.default_rng(42)
    for p in range(1, 9):
        for n in (1, 2, 5):
            knots = [0.0] * (p + 1) + [e / n for e in range(1, n)] + [1.0] * (p + 1)
            grev = [sum(knots[i + 1:i + p + 1]) / p for i in range(n + p)]
            for x in rng.uniform(0, 1, 20):
                _, f, v = eval_basis(p, n, x)
                assert np.all(v >= -1e-14)
                assert abs(v.sum() - 1.0) < 1e-13
                assert abs(sum(grev[f + k] * v[k] for k in range(p + 1)) - x) < 1e-12
                h = 1e-6
                if 2 * h < x < 1 - 2 * h:
                    _, fd_, d = eval_basis(p, n, x, deriv=1)
                    _, fp, vp = eval_basis(p, n, x + h)
                    _, fm, vm = eval_basis(p, n, x - h)
                    if fp == f and fm == f and fd_ == f:
                        assert np.allclose(d, (vp - vm) / (2 * h), rtol=5e-5, atol=1e-4)


def test_gram_frozen():  # test_spline.cpp:186-210
    m = gram(1, 1)
    assert np.allclose(m, [[1 / 3, 1 / 6], [1 / 6, 1 / 3]])
    k = gram(1, 1, deriv=1)
    assert np.allclose(k, [[1, -1], [-1, 1]])
    assert np.abs(gram(2, 1) - np.array([[6, 3, 1], [3, 4, 3], [1, 3, 6]]) / 30.0).max() < 1e-14
    k2 = 2.0 / 3.0 * np.array([[2, -1, -1], [-1, 2, -1], [-1, -1, 2]])
    assert np.abs(gram(2, 1, deriv=1) - k2).max() < 1e-14


def test_gram_against_finer_quadrature():  # test_spline.cpp:212-251
    for p in (2, 3, 4):
        n = 4
        m, k = gram(p, n, 1, 0), gram(p, n, 1, 0, deriv=1)
        dim = m.shape[0]
        m2, k2 = np.zeros((dim, dim)), np.zeros((dim, dim))
        _, xs, ws = gauss_legendre(2 * (p + 1))
        for e in range(n):
            for x0, w0 in zip(xs, ws):
                x, w = (e + x0) / n, w0 / n
                _, f, v = eval_basis(p, n, x, le=1)
                _, _, d = eval_basis(p, n, x, deriv=1, le=1)
                for a in range(p + 1):
                    ra = f + a - 1
                    if ra < 0 or ra >= dim:
                        continue
                    for b in range(p + 1):
                        rb = f + b - 1
                        if rb < 0 or rb >= dim:
                            continue
                        m2[ra, rb] += w * v[a] * v[b]
                        k2[ra, rb] += w * d[a] * d[b]
        assert np.abs(m - m2).max() < 1e-13
        assert np.abs(k - k2).max() < 1e-11
        assert np.linalg.eigvalsh(m)[0] > 0 and np.linalg.eigvalsh(k)[0] > -1e-12


def test_two_scale_frozen():  # test_spline.cpp:253-269
    assert np.abs(two_scale(1, 1) - np.array([[1, 0], [0.5, 0.5], [0, 1]])).max() < 1e-15
    e2 = np.array([[1, 0, 0], [0.5, 0.5, 0], [0, 0.5, 0.5], [0, 0, 1]])
    assert np.abs(two_scale(2, 1) - e2).max() < 1e-15


def _spline_value(p, n, le, re, c, x):
    _, f, v = eval_basis(p, n, x)
    dim = n + p - le - re
    s = 0.0
    for k in range(p + 1):
        r = f + k - le
        if 0 <= r < dim:
            s += c[r] * v[k]
    return s


def test_two_scale_reproduces_coarse_functions():  # test_spline.cpp:271-309
    rng = np.random.default_rng(7)
    for p in (1, 2, 3, 4):
        for n in (1, 2, 4):
            for le, re in ((0, 0), (1, 1), (1, 0)):
                P = two_scale(p, n, le, re)
                assert P.shape == (2 * n + p - le - re, n + p - le - re)
                c = rng.standard_normal(P.shape[1])
                f = P @ c
                for t in range(41):
                    x = t / 40
                    assert abs(_spline_value(p, 2 * n, le, re, f, x) - _spline_value(p, n, le, re, c, x)) < 1e-12
                if le == 0 and re == 0:
                    assert np.abs(P.sum(axis=1) - 1.0).max() < 1e-13


def test_gen_eig():  # test_spline.cpp:311-338
    rng = np.random.default_rng(3)
    n = 12
    a, b = rng.standard_normal((n, n)), rng.standard_normal((n, n))
    K = a.T @ a
    M = b.T @ b + np.eye(n)
    lam, V = np.zeros(n), np.zeros(n * n)
    Kf, Mf = np.asfortranarray(K), np.asfortranarray(M)
    assert N.host_lib().pmgh_gen_eig(n, Kf.ctypes.data_as(N._dp), Mf.ctypes.data_as(N._dp), lam.ctypes.data_as(N._dp),
                                     V.ctypes.data_as(N._dp)) == 0
    V = V.reshape(n, n).T
    assert np.all(np.diff(lam) >= -1e-14) and lam[0] > -1e-10
    assert np.abs(K @ V - M @ V @ np.diag(lam)).max() < 1e-9
    assert np.abs(V.T @ M @ V - np.eye(n)).max() < 1e-10
    # cross-check with LAPACK (scipy): same spectrum
    assert np.abs(lam - sla.eigh(K, M, eigvals_only=True)).max() < 1e-9 * lam.max()
    sing = np.zeros((2, 2))
    sing[0, 0] = 1.0
    eye = np.eye(2)
    out = np.zeros(4)
    assert N.host_lib().pmgh_gen_eig(2, eye.ctypes.data_as(N._dp), sing.ctypes.data_as(N._dp), out.ctypes.data_as(N._dp),
                                     out.ctypes.data_as(N._dp)) == N.PMG_ERR_DEFINITENESS


# ---------------------------------------------------------------- test_assembly.cpp
def _kron_sum(p, n, dim):
    K, M = gram(p, n, 1, 1, deriv=1), gram(p, n, 1, 1)
    if dim == 2:
        return np.kron(M, K) + np.kron(K, M)
    return np.kron(np.kron(M, M), K) + np.kron(np.kron(M, K), M) + np.kron(np.kron(K, M), M)


@pytest.mark.parametrize("p", [1, 2, 3])
def test_unit_square_stiffness_is_tensor_sum(p):  # test_assembly.cpp:112-128
    h = Hierarchy("unit_square_D", p, 2, n0=1)
    A = global_matrix(h, 2).toarray()
    oracle = _kron_sum(p, 4, 2)
    assert np.abs(A - oracle).max() < 1e-12 * np.abs(oracle).max()


def test_unit_cube_stiffness_is_tensor_sum():  # test_assembly.cpp:148-164
    h = Hierarchy("unit_grid(1,1,1)", 2, 1, n0=1)
    A = global_matrix(h, 1).toarray()
    oracle = _kron_sum(2, 2, 3)
    assert np.abs(A - oracle).max() < 1e-12 * np.abs(oracle).max()


def test_patch_stiffness_annihilates_constants():  # test_assembly.cpp:166-172
    """The free (un-eliminated) patch block maps constants to zero: every
    row of the raw band sums to 0 over the columns inside the lattice."""
    for name, p, n0 in [("lshape", 3, 1), ("c4", 3, 2), ("c2", 4, 2)]:
        h = Hierarchy(name, p, 2, n0=n0)
        band = h.band(2)
        ext = h.extent(2)
        lat = np.arange(ext ** h.dim)
        coords = [(lat // ext ** a) % ext for a in range(h.dim)]
        for k in range(h.num_patches):
            s = np.zeros(lat.size)
            scale = np.zeros(lat.size)
            for o, d in enumerate(band_offsets(h.dim, p)):
                ok = np.ones(lat.size, dtype=bool)
                for a in range(h.dim):
                    ok &= (coords[a] + d[a] >= 0) & (coords[a] + d[a] < ext)
                s += np.where(ok, band[k, o], 0.0)
                scale += np.abs(band[k, o])
            assert np.abs(s).max() < 1e-12 * scale.max()


def test_load_vector_kat():  # test_assembly.cpp:205-210
    # p = 1, n = 2, f = 1 on the unit square: the interior hat integrates to 1/4
    h = Hierarchy("unit_square_D", 1, 1, n0=1, rhs="one")
    r = h.rhs()
    assert r.size == 1 and r[0] == pytest.approx(0.25, abs=1e-15)


def test_stored_entries_bookkeeping():  # test_harness.cpp:111-128
    for p, n, d, k in [(2, 4, 2, 3), (3, 2, 3, 2), (4, 8, 2, 1)]:
        ext = n + p
        pairs = sum(min(i + p, ext - 1) - max(i - p, 0) + 1 for i in range(ext))
        assert N.host_lib().pmgh_stored_entries(p, n, d, k) == pairs ** d * k
    h = Hierarchy("lshape", 2, 2, n0=1)
    band = h.band(2)
    nz = sum(int(np.count_nonzero(np.abs(band[k]) > 0)) for k in range(h.num_patches))
    assert nz <= h.stored_entries(2)


def test_degenerate_geometry_and_config_errors():  # test_assembly.cpp:297-310, harness validation
    with pytest.raises(ConfigError):
        Hierarchy("no_such_domain", 2, 2)
    with pytest.raises(ConfigError):
        Hierarchy("lshape", 2, 0)
    with pytest.raises(DecompositionError):
        Hierarchy("unit_square_N", 2, 1, n0=1)  # singular coarse matrix (multigrid.cpp:38-48)


# ---------------------------------------------------------------- topology
def test_dof_counts_match_the_lattice_formula():
    for name, p, dirichlet_axes in [("c1", 2, (0, 1)), ("c2", 4, (0, 1)), ("c4", 3, (0,)), ("c5", 3, (0,))]:
        h = Hierarchy(name, p, 2, n0=2)
        k = {"c1": (2, 2), "c2": (4, 4), "c4": (2, 2, 2), "c5": (4, 4, 2)}[name]
        n = h.elements(2)
        expect = 1
        for a, ka in enumerate(k):
            cnt = ka * (n + p - 1) + 1
            if a in dirichlet_axes:
                cnt -= 2
            expect *= cnt
        assert h.num_dofs(2) == expect


def test_pieces_partition_the_dofs():  # test_topology.cpp:342-440, SPEC "Partition"
    for name, p, lv in [("lshape", 2, 2), ("fichera", 2, 2), ("c4", 3, 2), ("two_squares_flipped_D", 3, 2)]:
        h = Hierarchy(name, p, lv, n0=1 if name != "c4" else 2)
        for level in range(h.num_levels):
            seen = np.zeros(h.num_dofs(level), dtype=int)
            for pc in h.pieces(level):
                d = np.ctypeslib.as_array(pc.dofs, shape=(pc.ndofs,))
                seen[d] += 1
            assert np.all(seen == 1), (name, level)


def test_fichera_topology_and_vertex_scalars():  # test_topology.cpp:196-202, test_smoother.cpp:298-313
    h = Hierarchy("fichera", 2, 2, n0=1)
    assert len(h.interfaces()) == 9
    for level in (1, 2):
        hh = 1.0 / h.elements(level)
        verts = [pc for pc in h.pieces(level) if pc.kind == N.PIECE_VERTEX]
        assert verts and all(pc.scalar == hh / 2 for pc in verts)


def test_flipped_interface_orientation():  # test_topology.cpp:180-194
    h = Hierarchy("two_squares_flipped_D", 2, 1, n0=1)
    ifc = h.interfaces()
    assert len(ifc) == 1 and ifc[0][4] == 1


def test_baseline_generators_are_seeded_and_matching():
    a = Hierarchy("c4", 3, 1, n0=2, seed=42)
    b = Hierarchy("c4", 3, 1, n0=2, seed=42)
    c = Hierarchy("c4", 3, 1, n0=2, seed=43)
    assert np.array_equal(a.band(1), b.band(1)) and np.array_equal(a.rhs(), b.rhs())
    assert not np.array_equal(a.band(1), c.band(1))
    # every interior interface matched: 2x2x2 patches -> 12 interfaces
    assert len(a.interfaces()) == 12
    h2 = Hierarchy("c2", 4, 1, n0=2)
    assert len(h2.interfaces()) == 24


def test_gen_eig_cross_check_on_fd_payloads():
    """FD payload of an interior piece: V^T M V = I and K V = M V diag(lambda)
    for the piece's univariate spaces (spline.cpp:206-222), LAPACK cross-check."""
    h = Hierarchy("unit_square_D", 3, 3, n0=1)
    pc = [p for p in h.pieces(3) if p.kind == N.PIECE_INTERIOR][0]
    m = pc.dims[0]
    V = np.ctypeslib.as_array(pc.V[0], shape=(m * m,)).reshape(m, m).T
    K, M = gram(3, 8, 1, 1, deriv=1), gram(3, 8, 1, 1)
    assert np.abs(V.T @ M @ V - np.eye(m)).max() < 1e-10
    lam = np.diag(V.T @ K @ V)
    assert np.abs(np.sort(lam) - sla.eigh(K, M, eigvals_only=True)).max() < 1e-9 * lam.max()


def test_device_assembly_descriptor():
    """pmgh_build_ex(PMGH_DEVICE_ASSEMBLY): levels >= 1 carry no host band and
    name PMG_BAND_ASSEMBLE; the patch geometry is described for the device;
    host-only consumers refuse it loudly."""
    from paper_1804_02539_b200 import _native as N
    h = Hierarchy("c4", 3, 2, n0=2, assembly="device")
    hh = Hierarchy("c4", 3, 2, n0=2)
    assert h.desc.levels[0].band_format == N.PMG_BAND_TENSOR
    for l in range(1, h.num_levels):
        assert h.desc.levels[l].band_format == N.PMG_BAND_ASSEMBLE
        assert not h.desc.levels[l].band
        with pytest.raises(ValueError):
            h.band(l)
    assert np.array_equal(h.band(0), hh.band(0))
    g = h.desc.geometry
    assert g
    for k in range(h.num_patches):
        assert list(g[k].degree)[:3] == [1, 1, 1] and list(g[k].elements)[:3] == [1, 1, 1]
        assert np.isfinite(g[k].ctrl[0])
    import oracle
    with pytest.raises(Exception):
        oracle.Oracle(h)
    assert h.assemble_seconds() < hh.assemble_seconds()


def test_rhs_kind_resolution_and_zero_source():
    """pmgh_resolve_rhs_kind names the source PMGH_RHS_DEFAULT stands for (what
    pmg_assemble_load is given); the zero source skips the quadrature loop."""
    from paper_1804_02539_b200 import _native as N
    from paper_1804_02539_b200.hierarchy import RHS_KINDS
    lib = N.host_lib()
    assert lib.pmgh_resolve_rhs_kind(b"c1", 2, 0) == RHS_KINDS["sine_pi"]
    for dom in (b"c2", b"c5", b"jitter(2,2,1)"):
        assert lib.pmgh_resolve_rhs_kind(dom, 3, 0) == RHS_KINDS["random_nodes"]
    assert lib.pmgh_resolve_rhs_kind(b"lshape", 2, 0) == RHS_KINDS["sine2d"]
    assert lib.pmgh_resolve_rhs_kind(b"fichera", 3, 0) == RHS_KINDS["sine3d"]
    assert lib.pmgh_resolve_rhs_kind(b"fichera", 3, RHS_KINDS["one"]) == RHS_KINDS["one"]
    h = Hierarchy("c4", 3, 2, n0=2, rhs="zero")
    assert h.rhs().shape == (h.num_dofs(h.finest_level),) and not h.rhs().any()


def test_kronecker_levels_keep_the_host_band():
    """operator='kronecker' marks levels >= 1 PMG_BAND_KRONECKER for the device
    and leaves the assembled band in the descriptor for the CPU checker: the
    oracle runs on it unchanged."""
    from paper_1804_02539_b200 import _native as N
    import oracle
    hb = Hierarchy("c3", 3, 3, n0=2)
    hk = Hierarchy("c3", 3, 3, n0=2, operator="kronecker")
    assert hk.desc.levels[0].band_format == N.PMG_BAND_TENSOR
    for level in range(1, hk.num_levels):
        assert hk.desc.levels[level].band_format == N.PMG_BAND_KRONECKER
        assert np.array_equal(hk.band(level), hb.band(level))
    ub, hist_b, _, _ = oracle.Oracle(hb).pcg_solve(hb.rhs())
    uk, hist_k, _, _ = oracle.Oracle(hk).pcg_solve(hk.rhs())
    assert np.array_equal(ub, uk) and np.array_equal(hist_b, hist_k)
