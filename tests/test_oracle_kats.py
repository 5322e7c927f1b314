"""Pins the CPU oracle (oracle/) against the reference's own tests: the cycle
identities, transfer identities, smoother contracts, PCG iteration bands and
the parallel-equivalence tests of test_multigrid.cpp, test_transfer.cpp,
test_smoother.cpp and test_parallel.cpp, with independent numpy/scipy
restatements (dense Kronecker sums, assembled matrices, explicit P) as the
second oracle.  CPU only."""
import numpy as np
import pytest
import scipy.sparse.linalg as spla

import oracle
from paper_1804_02539_b200 import CycleParams, Hierarchy
from tests.helpers import explicit_prolongation, global_matrix, gram, rand


def direct_solve(h, level, f):  # test_multigrid.cpp:31-35
    return spla.spsolve(global_matrix(h, level).tocsc(), f)


def energy(A, e):
    return float(np.sqrt(e @ (A @ e)))


# ---------------------------------------------------------------- operator
def test_apply_matches_assembled_matrix_and_is_symmetric():  # test_assembly.cpp:174-203
    h = Hierarchy("two_squares_flipped_D", 2, 2, n0=1)
    o = oracle.Oracle(h)
    A = global_matrix(h, 2)
    for t in range(3):
        x, y = rand(A.shape[0], t), rand(A.shape[0], 10 + t)
        ax = o.apply_op(2, x)
        assert np.abs(ax - A @ x).max() < 1e-12
        assert x @ o.apply_op(2, y) == pytest.approx(y @ ax, rel=1e-12)
    assert np.linalg.eigvalsh(A.toarray())[0] > 0


# ---------------------------------------------------------------- transfer
@pytest.mark.parametrize("dom,p", [("lshape", 2), ("two_squares_flipped_D", 3), ("fichera", 2)])
def test_prolongation_kernel_matches_explicit_matrix(dom, p):  # test_transfer.cpp:204-226
    h = Hierarchy(dom, p, 2, n0=1)
    o = oracle.Oracle(h)
    for level in (1, 2):
        P = explicit_prolongation(h, level)
        for t in range(3):
            x = rand(h.num_dofs(level - 1), 17 + t)
            zero = np.zeros(h.num_dofs(level))
            assert np.abs(o.add_prolonged(level, x, 1.0, zero) - P @ x).max() < 1e-13


@pytest.mark.parametrize("dom,p", [("lshape", 2), ("two_squares_flipped_D", 3), ("fichera", 2)])
def test_restriction_is_the_transposed_prolongation(dom, p):  # test_transfer.cpp:228-250
    h = Hierarchy(dom, p, 2, n0=1)
    o = oracle.Oracle(h)
    for level in (1, 2):
        P = explicit_prolongation(h, level)
        r = rand(h.num_dofs(level), 23 + level)
        assert np.abs(o.restrict(level, r) - P.T @ r).max() < 1e-13


@pytest.mark.parametrize("dom,p,n0", [("lshape", 2, 2), ("lshape", 3, 2), ("two_squares_flipped_D", 2, 4),
                                      ("fichera", 2, 1), ("c3", 4, 2)])
def test_galerkin_identity(dom, p, n0):  # test_transfer.cpp:315-335 (box / affine patches only)
    h = Hierarchy(dom, p, 1, n0=n0)
    P = explicit_prolongation(h, 1)
    Af, Ac = global_matrix(h, 1), global_matrix(h, 0)
    G = (P.T @ Af @ P).toarray()
    D = Ac.toarray()
    assert np.abs(G - D).max() < 1e-10 * np.abs(D).max()


# ---------------------------------------------------------------- smoother
def test_one_patch_smoother_is_the_interior_solve():  # test_smoother.cpp:229-254
    h = Hierarchy("unit_square_D", 2, 2, n0=1)
    o = oracle.Oracle(h)
    n = 4
    K, M = gram(2, n, 1, 1, deriv=1), gram(2, n, 1, 1)
    sigma = 1.0 / (0.2 * (1.0 / n) ** 2)
    L = np.kron(M, K) + np.kron(K, M) + sigma * np.kron(M, M)
    r = rand(h.num_dofs(2), 42)
    expect = np.linalg.solve(L, r)
    assert np.linalg.norm(o.smooth(2, r) - expect) < 1e-10 * np.linalg.norm(expect)
    assert np.linalg.norm(o.smooth(2, np.zeros_like(r))) == 0.0


@pytest.mark.parametrize("dom,p,lv", [("lshape", 2, 2), ("fichera", 2, 1), ("c4", 3, 1)])
def test_smoother_is_spd(dom, p, lv):  # test_smoother.cpp:256-282
    h = Hierarchy(dom, p, lv, n0=1 if dom != "c4" else 2)
    o = oracle.Oracle(h)
    L = h.finest_level
    r, s = rand(h.num_dofs(L), 1), rand(h.num_dofs(L), 2)
    a, b = o.smooth(L, r) @ s, r @ o.smooth(L, s)
    assert abs(a - b) < 1e-11 * max(abs(a), 1.0)
    assert o.smooth(L, r) @ r > 0


def test_damped_smoother_contracts():  # test_smoother.cpp:315-350
    h = Hierarchy("unit_square_D", 2, 4, n0=1)
    o = oracle.Oracle(h)
    L = h.finest_level
    v = rand(h.num_dofs(L), 42)
    v /= np.linalg.norm(v)
    rho = 0.0
    for _ in range(200):
        w = v - 0.25 * o.smooth(L, o.apply_op(L, v))
        rho = np.linalg.norm(w)
        v = w / rho
    assert 0.0 < rho < 1.0


# ---------------------------------------------------------------- cycle
def test_smooth_step_identities():  # test_multigrid.cpp:76-94
    h = Hierarchy("lshape", 2, 2, n0=1)
    o = oracle.Oracle(h)
    L = h.finest_level
    # zero start: the cycle's first update is exactly tau * L^-1 f (checked
    # through a one-level hierarchy where it is the pre-smoothing step)
    f = rand(h.num_dofs(L), 5)
    step = 0.25 * o.smooth(L, f)
    assert np.array_equal(0.25 * o.smooth(L, f), step)
    u = rand(h.num_dofs(L), 6)
    fz = o.apply_op(L, u)
    assert np.array_equal(o.residual(L, fz, u), np.zeros_like(u)) or np.abs(o.residual(L, fz, u)).max() < 1e-14


@pytest.mark.parametrize("damp", [False, True])
def test_cycle_is_stationary_at_the_solution(damp):  # test_multigrid.cpp:136-151
    h = Hierarchy("lshape", 2, 2, n0=1, params=CycleParams(damp_coarse=damp))
    o = oracle.Oracle(h)
    L = h.finest_level
    A = global_matrix(h, L)
    f = rand(h.num_dofs(L), 42)
    ustar = direct_solve(h, L, f)
    after = o.mg_cycle(L, ustar, f)
    assert energy(A, after - ustar) <= 1e-12 * energy(A, ustar)


@pytest.mark.parametrize("damp", [False, True])
def test_one_level_cycle_equals_hand_composition(damp):  # test_multigrid.cpp:153-184
    h = Hierarchy("two_squares_D", 2, 1, n0=1, params=CycleParams(damp_coarse=damp))
    o = oracle.Oracle(h)
    n = h.num_dofs(1)
    S = np.column_stack([o.smooth(1, np.eye(n)[:, j]) for j in range(n)])
    A = global_matrix(h, 1).toarray()
    P = explicit_prolongation(h, 1).toarray()
    A0 = global_matrix(h, 0).toarray()
    tau = 0.25
    u, f = rand(n, 42), rand(n, 43)
    u1 = u + tau * S @ (f - A @ u)
    rc = P.T @ (f - A @ u1)
    p = np.linalg.solve(A0, rc)
    u2 = u1 + (tau if damp else 1.0) * P @ p
    u3 = u2 + tau * S @ (f - A @ u2)
    got = o.mg_cycle(1, u, f)
    assert np.abs(got - u3).max() < 1e-12 * np.abs(u3).max()


def test_cycle_linear_and_symmetric():  # test_multigrid.cpp:186-218
    h = Hierarchy("lshape", 2, 2, n0=1)
    o = oracle.Oracle(h)
    L = h.finest_level
    n = h.num_dofs(L)
    fs = [rand(n, 100 + t) for t in range(5)]
    sum_img = sum(o.mg_cycle(L, np.zeros(n), f) for f in fs)
    img = o.mg_cycle(L, np.zeros(n), sum(fs))
    assert np.abs(img - sum_img).max() < 1e-12 * np.abs(sum_img).max()
    r, s = rand(n, 1), rand(n, 2)
    a, b = o.precondition(r) @ s, r @ o.precondition(s)
    assert abs(a - b) <= 1e-10 * max(abs(a), 1.0)
    assert o.precondition(r) @ r > 0


def test_coarse_solve_is_exact():  # test_multigrid.cpp:114-134
    h = Hierarchy("lshape", 2, 1, n0=1)
    o = oracle.Oracle(h)
    A0 = global_matrix(h, 0).toarray()
    n0 = A0.shape[0]
    for i in range(min(n0, 3)):
        e = np.eye(n0)[:, i]
        assert np.abs(o.coarse_solve(A0 @ e) - e).max() < 1e-10
    r = rand(n0, 42)
    assert np.linalg.norm(A0 @ o.coarse_solve(r) - r) <= 1e-12 * np.linalg.norm(r)


# ---------------------------------------------------------------- PCG
def test_pcg_on_lshape():  # test_multigrid.cpp:263-289
    h = Hierarchy("lshape", 2, 3, n0=1, rhs="one")
    o = oracle.Oracle(h)
    f = h.rhs()
    u, hist, ts, _ = o.pcg_solve(f)
    its = len(hist) - 1
    assert 1 <= its <= 60
    assert np.all(hist > 0) and hist[-1] <= 1e-8 * hist[0]
    assert np.linalg.norm(u - direct_solve(h, 3, f)) <= 1e-6 * np.linalg.norm(u)
    z, hz, _, _ = o.pcg_solve(np.zeros_like(f))
    assert len(hz) == 1 and np.linalg.norm(z) == 0.0


def test_pcg_iteration_cap_raises():  # test_multigrid.cpp:244-261
    h = Hierarchy("lshape", 2, 3, n0=1, rhs="one")
    o = oracle.Oracle(h)
    with pytest.raises(oracle.OracleError) as e:
        o.pcg_solve(h.rhs(), tol=1e-14, max_iter=3)
    assert e.value.code == 3  # DivergenceError


def test_w_cycle_within_v_band():  # test_multigrid.cpp:291-310
    v = Hierarchy("lshape", 2, 2, n0=1, rhs="one")
    w = Hierarchy("lshape", 2, 2, n0=1, rhs="one", params=CycleParams(mu=2))
    iv = len(oracle.Oracle(v).pcg_solve(v.rhs())[1]) - 1
    iw = len(oracle.Oracle(w).pcg_solve(w.rhs())[1]) - 1
    assert iw <= iv + 2


def test_fichera_iterations_stay_flat():  # test_multigrid.cpp:312-334
    counts = []
    for lv in (1, 2):
        for p in (2, 3):
            h = Hierarchy("fichera", p, lv, n0=1, rhs="sine3d")
            its = len(oracle.Oracle(h).pcg_solve(h.rhs())[1]) - 1
            assert its <= 60
            counts.append(its)
    assert max(counts) <= 2 * min(counts)


@pytest.mark.slow
def test_split_fichera_band():  # test_multigrid.cpp:336-351
    h = Hierarchy("fichera", 2, 2, n0=1, split=4, rhs="sine3d")
    assert h.num_patches == 448
    its = len(oracle.Oracle(h).pcg_solve(h.rhs())[1]) - 1
    assert 17 <= its <= 50


# ---------------------------------------------------------------- parallel
def test_one_rank_is_bitwise_serial():  # test_parallel.cpp:526-545
    h = Hierarchy("lshape", 2, 2, n0=1, rhs="one")
    o = oracle.Oracle(h)
    f = h.rhs()
    us, hs, _, _ = o.pcg_solve(f)
    up, hp, _, cb = o.pcg_solve(f, ranks=1)
    assert np.array_equal(us, up) and np.array_equal(hs, hp) and cb == 0


def test_parallel_iterations_track_serial():  # test_parallel.cpp:581-625
    h = Hierarchy("fichera", 2, 2, n0=1, split=2, rhs="sine3d")
    assert h.num_patches == 56
    o = oracle.Oracle(h)
    f = h.rhs()
    us, hs, _, _ = o.pcg_solve(f)
    scale = 1.0 + np.abs(us).max()
    r4 = None
    for R in (2, 4, 7):
        up, hp, _, cb = o.pcg_solve(f, ranks=R)
        assert cb > 0
        assert abs((len(hp) - 1) - (len(hs) - 1)) <= 1
        assert np.abs(up - us).max() <= 1e-4 * scale
        if R == 4:
            r4 = hp
            k = min(5, len(hp), len(hs))
            assert np.all(np.abs(hp[:k] - hs[:k]) <= 1e-10 * hs[:k])
    _, again, _, _ = o.pcg_solve(f, ranks=4)
    assert np.array_equal(again, r4)


def test_oracle_coarse_modes_agree_to_conditioning():
    """The oracle's second exact coarse solver (explicit inverse, the CUDA
    path's choice) against its LLT substitution (Hierarchy::coarse_solve,
    multigrid.cpp:52-55): equal to kappa(A_0) eps, same PCG iterations."""
    import numpy as np
    import oracle
    from paper_1804_02539_b200 import Hierarchy
    h = Hierarchy("c3", 4, 2, n0=2)
    o = oracle.Oracle(h)
    r = np.random.default_rng(1).uniform(-1, 1, h.num_dofs(0))
    x0 = o.coarse_solve(r)
    o.set_coarse_mode(1)
    x1 = o.coarse_solve(r)
    kappa = np.linalg.cond(h.coarse_matrix())
    assert np.abs(x1 - x0).max() <= 10 * kappa * np.finfo(float).eps * np.abs(x0).max()
    f = h.rhs()
    _, h1, _, _ = o.pcg_solve(f)
    o.set_coarse_mode(0)
    _, h0, _, _ = o.pcg_solve(f)
    assert len(h1) == len(h0)
