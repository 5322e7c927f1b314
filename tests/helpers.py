"""Independent numpy/scipy restatements used by the CPU tests as second
oracles (dense Kronecker products, assembled global matrices, explicit
prolongation matrices), mirroring the oracles of the reference tests
(test_assembly.cpp:112-164, test_transfer.cpp:204-250, test_multigrid.cpp:31-35)."""
import ctypes as C

import numpy as np
import scipy.sparse as sp

from paper_1804_02539_b200 import _native as N


def gram(p, n, le=0, re=0, deriv=0):
    lib = N.host_lib()
    dim = C.c_int()
    assert lib.pmgh_gram(p, n, le, re, deriv, C.byref(dim), None) == 0
    out = np.empty(dim.value * dim.value)
    assert lib.pmgh_gram(p, n, le, re, deriv, C.byref(dim), out.ctypes.data_as(N._dp)) == 0
    return out.reshape(dim.value, dim.value).T.copy()


def two_scale(p, n, le=0, re=0):
    lib = N.host_lib()
    fd, cd = C.c_int(), C.c_int()
    assert lib.pmgh_two_scale(p, n, le, re, C.byref(fd), C.byref(cd), None) == 0
    out = np.empty(fd.value * cd.value)
    assert lib.pmgh_two_scale(p, n, le, re, C.byref(fd), C.byref(cd), out.ctypes.data_as(N._dp)) == 0
    return out.reshape(cd.value, fd.value).T.copy()


def eval_basis(p, n, x, deriv=0, le=0, re=0):
    lib = N.host_lib()
    first = C.c_int()
    vals = np.zeros(p + 1)
    rc = lib.pmgh_eval_basis(p, n, le, re, x, deriv, C.byref(first), vals.ctypes.data_as(N._dp))
    return rc, first.value, vals


def gauss_legendre(q):
    nodes, weights = np.zeros(q), np.zeros(q)
    rc = N.host_lib().pmgh_gauss_legendre(q, nodes.ctypes.data_as(N._dp), weights.ctypes.data_as(N._dp))
    return rc, nodes, weights


def band_offsets(dim, p):
    w = 2 * p + 1
    offs = []
    for o in range(w ** dim):
        d = []
        for _ in range(dim):
            d.append(o % w - p)
            o //= w
        offs.append(d)
    return offs


def global_matrix(h, level):
    """The summed global stiffness (MultiPatchOperator::assemble_global,
    assembly.cpp:282-297) from the index-free band and l2g."""
    dim, p = h.dim, h.degree
    ext = h.extent(level)
    band = h.band(level)
    l2g = h.l2g(level)
    rows, cols, vals = [], [], []
    lat = np.arange(ext ** dim)
    coords = [(lat // ext ** a) % ext for a in range(dim)]
    for o, d in enumerate(band_offsets(dim, p)):
        ok = np.ones(lat.size, dtype=bool)
        col = np.zeros(lat.size, dtype=np.int64)
        for a in range(dim):
            ca = coords[a] + d[a]
            ok &= (ca >= 0) & (ca < ext)
            col += np.clip(ca, 0, ext - 1) * ext ** a
        for k in range(h.num_patches):
            g_r = l2g[k]
            g_c = l2g[k][col]
            m = ok & (g_r >= 0) & (g_c >= 0)
            rows.append(g_r[m])
            cols.append(g_c[m])
            vals.append(band[k, o][m])
    n = h.num_dofs(level)
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))), shape=(n, n))


def owner_patch(h, level):
    off, pat, _ = h.reps(level)
    return pat[off[:-1]]


def explicit_prolongation(h, level):
    """TransferOperator::explicit_matrix (transfer.cpp:93-141)."""
    dim = h.dim
    P1 = h.two_scale_dense(level)
    ext_f, ext_c = h.extent(level), h.extent(level - 1)
    Pk = P1
    for _ in range(dim - 1):
        Pk = np.kron(P1, Pk)  # axis 0 fastest
    l2g_f, l2g_c = h.l2g(level), h.l2g(level - 1)
    own = owner_patch(h, level)
    rows, cols, vals = [], [], []
    for k in range(h.num_patches):
        gf = l2g_f[k]
        mask = gf >= 0
        mask[mask] = own[gf[mask]] == k
        sub = Pk[mask]
        gc = l2g_c[k]
        cmask = gc >= 0
        sub = sub[:, cmask]
        r, c = np.nonzero(sub)
        rows.append(gf[mask][r])
        cols.append(gc[cmask][c])
        vals.append(sub[r, c])
    return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                         shape=(h.num_dofs(level), h.num_dofs(level - 1)))


def rand(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


# The driver runs `pytest -m gpu` under a 20-minute limit.  The default
# selection keeps every BASELINE family at full size and every kernel
# configuration; PMG_TEST_FULL=1 (scripts/gpu_round.sh) adds the remaining
# combinations (all five c3 degrees at full size, every FD configuration on
# every desk hierarchy, the full-c4 host-vs-device assembly comparison).
import os  # noqa: E402

FULL_MATRIX = os.environ.get("PMG_TEST_FULL") == "1"
