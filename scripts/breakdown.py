"""Per-level, per-kernel-class device time of one PCG solve (CUDA events around
every launch group; instrumented replay without CUDA graphs).

  python scripts/breakdown.py [config] [solves] [levels]
"""
import ctypes as C
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

from paper_1804_02539_b200 import _native as N  # noqa: E402
from paper_1804_02539_b200.backend import GpuBackend  # noqa: E402
from paper_1804_02539_b200.hierarchy import CONFIGS, Hierarchy  # noqa: E402

CLASSES = {0: "spmv", 1: "fd_interior", 2: "transfer", 3: "interface_pieces", 4: "vector_ops", 5: "coarse"}

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
solves = int(sys.argv[2]) if len(sys.argv) > 2 else 3
levels = int(sys.argv[3]) if len(sys.argv) > 3 else None
dom, p, n0, lv = CONFIGS[name]
h = Hierarchy(dom, p, lv if levels is None else levels, n0=n0)
b = GpuBackend(h)
lib = N.cuda_lib()
L = h.finest_level
f = b.to_distributed_owner(L, h.rhs())
u = b.zero_acc(L)
u, rep = b.pcg_solve_device(f, u=u)
b.synchronize()
t0 = time.perf_counter()
for _ in range(solves):
    u, rep = b.pcg_solve_device(f, u=u)
b.synchronize()
t_graph = (time.perf_counter() - t0) / solves * 1e3
lib.pmg_profile(b._ctx, 1)
t0 = time.perf_counter()
for _ in range(solves):
    u, rep = b.pcg_solve_device(f, u=u)
b.synchronize()
t_prof = (time.perf_counter() - t0) / solves * 1e3
lib.pmg_profile(b._ctx, 0)
rows = []
tot = 0.0
for cls, cname in CLASSES.items():
    for level in range(h.num_levels):
        n, ms, w = C.c_int64(), C.c_double(), C.c_double()
        lib.pmg_profile_read(b._ctx, cls, level, C.byref(n), C.byref(ms), C.byref(w))
        if n.value:
            rows.append({"class": cname, "level": level, "launch_groups": n.value / solves, "ms": ms.value / solves,
                         "work": w.value / solves})
            tot += ms.value / solves
print(f"{name}: {h.num_dofs(L)} dofs, {rep.iterations} iterations; wall ms/solve: graphs {t_graph:.2f}, "
      f"instrumented {t_prof:.2f}; summed kernel ms {tot:.2f}")
for r in sorted(rows, key=lambda r: -r["ms"]):
    extra = ""
    if r["class"] == "spmv" and r["ms"]:
        extra = f"  {r['work'] / (r['ms'] / 1e3) / 1e9:7.0f} GB/s"
    if r["class"] == "fd_interior" and r["ms"]:
        extra = f"  {r['work'] / (r['ms'] / 1e3) / 1e12:7.2f} TFLOP/s"
    print(f"{r['class']:>16s} L{r['level']}  {r['ms']:8.3f} ms  {100 * r['ms'] / tot:5.1f}%  "
          f"{r['launch_groups']:6.1f} groups{extra}")
Path("gpurun_out").mkdir(exist_ok=True)
Path(f"gpurun_out/breakdown_{name}.json").write_text(json.dumps(
    {"config": name, "t_graph_ms": t_graph, "t_instrumented_ms": t_prof, "rows": rows}, indent=1))
