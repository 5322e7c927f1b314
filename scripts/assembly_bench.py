"""Stiffness assembly: host (libpmg_host, all cores) vs device (assembly.cu)
for BASELINE configs.  Prints one JSON line per config."""
import json
import os
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402

from paper_1804_02539_b200 import baseline_hierarchy  # noqa: E402
from paper_1804_02539_b200.backend import GpuBackend  # noqa: E402
from paper_1804_02539_b200.hierarchy import CONFIGS, Hierarchy  # noqa: E402

for name in sys.argv[1:] or ["c2", "c4"]:
    dom, p, n0, lv = CONFIGS[name]
    t0 = time.perf_counter()
    hh = baseline_hierarchy(name)
    t_host_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    hd = Hierarchy(dom, p, lv, n0=n0, assembly="device")
    t_dev_build = time.perf_counter() - t0
    bd = GpuBackend(hd)
    bh = GpuBackend(hh)
    rng = np.random.default_rng(1)
    L = hh.finest_level
    u = rng.uniform(-1, 1, hh.num_dofs(L))
    yh = bh.gather_global(L, bh.apply_op(L, bh.to_accumulated(L, u)))
    yd = bd.gather_global(L, bd.apply_op(L, bd.to_accumulated(L, u)))
    entries = sum(hh.stored_entries(l) for l in range(1, hh.num_levels))
    print(json.dumps({
        "config": name, "band_entries_levels_ge1": entries,
        "host_assembly_s": hh.assemble_seconds(), "host_threads": os.cpu_count(),
        "host_build_total_s": t_host_build, "device_hierarchy_host_setup_s": t_dev_build,
        "device_assembly_s": bd.assembly_seconds(),
        "finest_apply_rel_diff": float(np.abs(yd - yh).max() / np.abs(yh).max()),
    }), flush=True)
