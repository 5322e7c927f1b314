"""Build the hierarchy of a BASELINE config and run N device-resident PCG
solves (graph-replayed), for ncu launch lists and captures.

  python scripts/solve_once.py [config] [solves] [levels]
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1804_02539_b200.backend import GpuBackend  # noqa: E402
from paper_1804_02539_b200.hierarchy import CONFIGS, Hierarchy  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
solves = int(sys.argv[2]) if len(sys.argv) > 2 else 1
levels = int(sys.argv[3]) if len(sys.argv) > 3 else None
dom, p, n0, lv = CONFIGS[name]
h = Hierarchy(dom, p, lv if levels is None else levels, n0=n0)
b = GpuBackend(h)
L = h.finest_level
f = b.to_distributed_owner(L, h.rhs())
for i in range(solves):
    t = time.perf_counter()
    u, rep = b.pcg_solve_device(f)
    print(f"solve {i}: {rep.iterations} iterations, {1e3 * (time.perf_counter() - t):.2f} ms wall")
