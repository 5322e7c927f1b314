"""Committed golden fixtures (tests/golden/*.npz, made by
tests/golden/make_golden.py from the KAT-pinned oracle).

CPU: the host setup (load vector) and the oracle still reproduce the frozen
answers, so any drift in either is caught against a version-controlled file.
GPU: the CUDA path, through the C ABI, meets the fixtures with the
north_star tolerances (identical PCG iteration counts, solution within 1e-10
relative, residual norms within 1e-10 ||r_k|| + floor ||r_0||; single
operators at 1e-13, the V-cycle preconditioner at 1e-11)."""
import glob
import os

import numpy as np
import pytest

from paper_1804_02539_b200 import Hierarchy

GOLDEN = sorted(glob.glob(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "*.npz")))
IDS = [os.path.basename(g)[:-4] for g in GOLDEN]


def rel(a, b):
    return np.abs(a - b).max() / max(np.abs(b).max(), 1e-300)


def load(path):
    g = dict(np.load(path))
    h = Hierarchy(str(g["domain"]), int(g["degree"]), int(g["levels"]), n0=int(g["n0"]), rhs=str(g["rhs"]))
    return g, h


def test_golden_set_present():
    assert len(GOLDEN) >= 7


@pytest.mark.parametrize("path", GOLDEN, ids=IDS)
def test_oracle_reproduces_golden(path):
    import oracle

    g, h = load(path)
    L = h.finest_level
    assert np.array_equal(h.rhs(), g["f"])
    o = oracle.Oracle(h)
    u, hist, _, _ = o.pcg_solve(g["f"])
    assert len(hist) - 1 == int(g["iterations"])
    assert rel(hist, g["history"]) < 1e-12
    assert rel(u, g["u"]) < 1e-12
    assert rel(o.apply_op(L, g["x_op"]), g["y_op"]) < 1e-13
    assert rel(o.smooth(L, g["r_smooth"]), g["z_smooth"]) < 1e-13
    assert rel(o.precondition(g["r_pre"]), g["z_pre"]) < 1e-12
    assert rel(o.restrict(L, g["r_restrict"]), g["c_restrict"]) < 1e-13


@pytest.mark.gpu
@pytest.mark.parametrize("path", GOLDEN, ids=IDS)
def test_gpu_meets_golden(path):
    from paper_1804_02539_b200.backend import GpuBackend

    g, h = load(path)
    L = h.finest_level
    b = GpuBackend(h)
    y = b.gather_global(L, b.apply_op(L, b.to_accumulated(L, g["x_op"])))
    assert rel(y, g["y_op"]) < 1e-13
    z = b.gather_global(L, b.smooth(L, b.to_distributed_owner(L, g["r_smooth"])))
    assert rel(z, g["z_smooth"]) < 1e-12
    z = b.gather_global(L, b.precondition(b.to_distributed_owner(L, g["r_pre"])))
    assert rel(z, g["z_pre"]) < 1e-11
    c = b.gather_global(L - 1, b.restrict_residual(L, b.to_distributed_owner(L, g["r_restrict"])))
    assert rel(c, g["c_restrict"]) < 1e-13
    u, rep = b.pcg_solve(g["f"])
    ref = g["history"]
    assert rep.iterations == int(g["iterations"])
    hist = np.array(rep.residual_history)
    assert np.all(np.abs(hist - ref) <= 1e-10 * ref + float(g["floor"]) * ref[0])
    assert rel(u, g["u"]) < 1e-10
