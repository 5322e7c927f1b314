"""One PCG solve of a BASELINE config on cuda:0 (for ncu launch lists)."""
import sys
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
f = b.to_distributed_owner(h.finest_level, h.rhs())
u = b.zero_acc(h.finest_level)
for _ in range(solves):
    u, rep = b.pcg_solve_device(f, u=u)
print(name, "iterations", rep.iterations, "launches", b.kernel_launches())
