"""Bitwise run-to-run determinism of the device path (a race shows up as a
changed bit).  Usage: python scripts/determinism.py [reps]"""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1804_02539_b200 import Hierarchy
from paper_1804_02539_b200.backend import GpuBackend, pcg_generic

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
bad = 0
for dom, p, lv, n0 in [("c2", 4, 5, 2), ("c1", 2, 5, 2), ("c4", 3, 3, 2), ("c3", 8, 5, 2), ("fichera", 2, 5, 1)]:
    h = Hierarchy(dom, p, lv, n0=n0)
    b = GpuBackend(h)
    L = h.finest_level
    f = h.rhs()
    rng = np.random.default_rng(0)
    u = rng.uniform(-1, 1, h.num_dofs(L))
    uacc = b.to_accumulated(L, u)
    fd = b.to_distributed_owner(L, f)
    y0 = b.apply_op(L, uacc).lattice()
    z0 = b.precondition(fd).lattice()
    s0, rep0 = b.pcg_solve(f)
    h0 = np.array(rep0.residual_history)
    for i in range(reps):
        y = b.apply_op(L, uacc).lattice()
        z = b.precondition(fd).lattice()
        s, rep = b.pcg_solve(f)
        hh = np.array(rep.residual_history)
        msg = []
        if not np.array_equal(y, y0):
            msg.append(f"apply_op differs at {np.flatnonzero(y != y0)[:5]}")
        if not np.array_equal(z, z0):
            msg.append(f"precondition differs ({np.count_nonzero(z != z0)} entries)")
        if rep.iterations != rep0.iterations or not np.array_equal(hh, h0) or not np.array_equal(s, s0):
            msg.append(f"pcg differs: its {rep.iterations} vs {rep0.iterations}")
        if msg:
            bad += 1
            print(dom, p, lv, "rep", i, "; ".join(msg), flush=True)
    hist = []
    pcg_generic(b, fd, 1e-8, 500, lambda r: b.precondition(r), hist)
    print(dom, p, lv, "its", rep0.iterations, "generic its", len(hist) - 1, flush=True)
    del b
print("DETERMINISM", "FAIL" if bad else "OK", bad)
