"""Generates the committed golden fixtures in tests/golden/*.npz.

Each fixture freezes, for one small hierarchy, the outputs of the CPU oracle
(oracle/, the restatement of the reference solve path pinned by
tests/test_oracle_kats.py and tests/test_setup_kats.py against the
reference's own known-answer tests):

  f, u, history        the seeded load vector, the PCG solution and the
                       residual-norm history of pcg_solve (multigrid.hpp:155-189)
  iterations           the PCG iteration count
  floor                the residual-history floor of tests/test_gpu_parity.py
                       (history_floor), frozen with the fixture
  x_op, y_op           apply_op(finest, x_op)          (operator.cpp:28-70)
  r_smooth, z_smooth   smooth(finest, r_smooth)        (smoother.cpp)
  r_pre, z_pre         precondition(r_pre)             (multigrid.hpp:143-153)
  r_restrict, c_restrict  restrict(finest, r)          (transfer.cpp)

The reference itself (C++20 + Eigen3) does not build in this image
(DESIGN.md), so the fixtures are oracle outputs; what they add over the live
oracle is a frozen, version-controlled answer that the GPU tests and any
future oracle change are held to.  Regenerate with
    python tests/golden/make_golden.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

# (name, domain, degree, levels, n0, rhs)
CASES = [
    ("lshape_p2_L3", "lshape", 2, 3, 1, "one"),
    ("two_squares_flipped_D_p3_L3", "two_squares_flipped_D", 3, 3, 1, "sine2d"),
    ("fichera_p2_L2", "fichera", 2, 2, 1, "sine3d"),
    ("c1_p2_L3", "c1", 2, 3, 2, "default"),
    ("c2_p4_L3", "c2", 4, 3, 2, "default"),
    ("c3_p6_L3", "c3", 6, 3, 2, "default"),
    ("c4_p3_L2", "c4", 3, 2, 2, "default"),
]
HERE = os.path.dirname(os.path.abspath(__file__))


def seeded(n, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def make(case):
    import oracle
    from paper_1804_02539_b200 import Hierarchy
    from tests.test_gpu_parity import history_floor

    name, dom, p, lv, n0, rhs = case
    h = Hierarchy(dom, p, lv, n0=n0, rhs=rhs)
    o = oracle.Oracle(h)
    L = h.finest_level
    n = h.num_dofs(L)
    f = h.rhs()
    u, hist, _, _ = o.pcg_solve(f)
    x_op, r_smooth, r_pre, r_restrict = (seeded(n, s) for s in (1, 2, 3, 4))
    out = dict(
        domain=dom, degree=p, levels=lv, n0=n0, rhs=rhs,
        f=f, u=u, history=hist, iterations=len(hist) - 1,
        floor=history_floor(h, o, f, hist),
        x_op=x_op, y_op=o.apply_op(L, x_op),
        r_smooth=r_smooth, z_smooth=o.smooth(L, r_smooth),
        r_pre=r_pre, z_pre=o.precondition(r_pre),
        r_restrict=r_restrict, c_restrict=o.restrict(L, r_restrict),
    )
    np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
    print(f"{name}: {n} dofs, {len(hist) - 1} iterations")


if __name__ == "__main__":
    for c in CASES:
        make(c)
