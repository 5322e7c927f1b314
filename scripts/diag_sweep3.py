"""Diagnose the 3D plane sweep against the 256-row kernel on one config:
python scripts/diag_sweep3.py dom p lv n0 min_ext"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1804_02539_b200 import Hierarchy  # noqa: E402
from paper_1804_02539_b200.backend import GpuBackend  # noqa: E402

dom, p, lv, n0, me = sys.argv[1], int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4]), sys.argv[5]
h = Hierarchy(dom, p, lv, n0=n0)
out = {}
for mode in (me, "0"):
    os.environ["PMG_SWEEP3D"] = mode
    b = GpuBackend(h)
    res = []
    for level in range(h.num_levels):
        u = np.random.default_rng(31 + level).uniform(-1, 1, h.num_dofs(level))
        ua = b.to_accumulated(level, u)
        y = b.apply_op(level, ua)
        res.append((y.lattice().copy(), b.dot(level, y, ua)))
    out[mode] = res
    del b
for level in range(h.num_levels):
    a, b_ = out[me][level][0], out["0"][level][0]
    d = np.abs(a - b_)
    ext = h.extent(level)
    print(f"level {level} ext {ext}: max|d| {d.max():.3e} max|y| {np.abs(b_).max():.3e}  dot {out[me][level][1]:.6e} vs {out['0'][level][1]:.6e}")
    if d.max() > 1e-10 * np.abs(b_).max():
        lat = d.reshape(h.num_patches, ext, ext, ext)  # [k][i2][i1][i0]
        bad = np.argwhere(lat > 1e-10 * np.abs(b_).max())
        print("  bad entries", len(bad), "first", bad[:10].tolist())
        planes = sorted(set(bad[:, 1].tolist()))
        print("  planes", planes[:40])
        print("  patches", sorted(set(bad[:, 0].tolist()))[:40])
