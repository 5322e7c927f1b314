"""One preconditioner application (V-cycle from zero) on a BASELINE config,
for kernel launch lists: python scripts/precond_once.py c2"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_1804_02539_b200 import baseline_hierarchy  # noqa: E402
from paper_1804_02539_b200.backend import GpuBackend  # noqa: E402

h = baseline_hierarchy(sys.argv[1] if len(sys.argv) > 1 else "c2")
b = GpuBackend(h)
r = b.to_distributed_owner(h.finest_level, h.rhs())
for _ in range(2):
    b.precondition(r)
b.synchronize() if hasattr(b, "synchronize") else None
