#!/usr/bin/env python
"""Benchmark of the PCG + V(1,1)-cycle solve path (BASELINE.json metric).

One step = one PCG solve (zero start, V(1,1) preconditioner, tol 1e-8) of the
workload on N GPUs.  Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl reference]

value   DOF x PCG iterations / s over all ranks, device-resident inputs
        (the per-iteration work is one V(1,1) cycle + one SpMV + 3 dots)
e2e     the same metric through pmg_pcg_solve from pinned host memory:
        global load vector H2D and global solution D2H inside every step
roofline  the band SpMV on the finest level, timed live with CUDA events on
        the launch stream; algorithmic bytes = 8 B per stored reference CSR
        entry + 8 B per lattice row for x, y (and f) -- SURVEY 8(d)
--impl reference  the CPU oracle (restatement of the reference solve path,
        oracle/) with all host threads, bounded samples of one PCG iteration.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

WORKLOADS = {
    "c1": "2D Poisson, 2x2 affine patches, p=2, 64^2 elements/patch (BASELINE config 1)",
    "c2": "2D Poisson, 4x4 sinusoidally perturbed patches, p=4, 256^2 elements/patch (BASELINE config 2)",
    "c3p2": "2D 4x4 patches, p=2, 128^2 elements/patch (BASELINE config 3)",
    "c3p3": "2D 4x4 patches, p=3, 128^2 elements/patch (BASELINE config 3)",
    "c3p4": "2D 4x4 patches, p=4, 128^2 elements/patch (BASELINE config 3)",
    "c3p6": "2D 4x4 patches, p=6, 128^2 elements/patch (BASELINE config 3)",
    "c3p8": "2D 4x4 patches, p=8, 128^2 elements/patch (BASELINE config 3)",
    "c4": "3D Poisson, 2x2x2 jittered trilinear patches, p=3, 64^3 elements/patch (BASELINE config 4)",
    "c5": "3D Poisson, 4x4x2 jittered trilinear patches, p=3, 64^3 elements/patch (BASELINE config 5)",
}
METRIC = "PCG-MG solve throughput: DOF x PCG iterations per second (one V(1,1) cycle + SpMV per iteration), fp64"
UNIT = "DOF*iter/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c2")
    ap.add_argument("--levels", type=int, default=None, help="override the refinement depth")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target length of the CPU sample")
    ap.add_argument("--assembly", default="host", choices=["host", "device"],
                    help="stiffness assembly of levels >= 1 (device: on the B200, DESIGN.md 3a; "
                         "no CPU baseline then, the oracle needs host bands)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi style sampling of SM clocks and throttle reasons (NVML)."""

    REASONS = {
        0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
        0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
        0x100: "display_clock_setting",
    }

    def __init__(self, device: int):
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(device)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nv = None

    def _run(self):
        while not self._stop.is_set():
            try:
                clk = self._nv.nvmlDeviceGetClockInfo(self._h, self._nv.NVML_CLOCK_SM)
                util = self._nv.nvmlDeviceGetUtilizationRates(self._h).gpu
                mask = self._nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append((clk, util))
                for bit, name in self.REASONS.items():
                    if mask & bit and bit != 0x1:
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.1)

    def __enter__(self):
        if self._nv:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._nv:
            self._t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons), "samples": 0}
        loaded = [c for c, u in self.samples if u > 0] or [c for c, _ in self.samples]
        return {"sm_mhz": statistics.median(loaded), "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def build_hierarchy(args, threads=None):
    from paper_1804_02539_b200.hierarchy import CONFIGS, Hierarchy
    dom, p, n0, lv = CONFIGS[args.config]
    if args.levels is not None:
        lv = args.levels
    return Hierarchy(dom, p, lv, n0=n0, seed=args.seed, threads=threads,
                     assembly=getattr(args, "assembly", "host"))


def workload_config(args, h, extra=None):
    L = h.finest_level
    cfg = {
        "workload": f"{args.config}: {WORKLOADS.get(args.config, args.config)}; PCG + V(1,1), tol 1e-8, zero start",
        "dofs": h.num_dofs(L), "levels": h.num_levels, "degree": h.degree, "patches": h.num_patches,
        "elements_per_patch_dir": h.elements(L), "coarsest_elements": h.elements(0),
        "stored_band_entries_finest": h.stored_entries(L),
        "l2": "inputs larger than L2 (finest band alone exceeds 126 MB)" if h.stored_entries(L) * 8 > 126e6
        else "inputs smaller than L2; no flush (solve is latency bound)",
    }
    if extra:
        cfg.update(extra)
    return cfg


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import numpy as np
    import oracle
    threads = os.cpu_count() or 1
    h = build_hierarchy(args, threads=threads)
    o = oracle.Oracle(h)
    f = h.rhs()
    ranks = max(1, min(threads, h.num_patches))
    n = h.num_dofs(h.finest_level)
    # one step = a bounded sample: one PCG iteration (initial preconditioner,
    # SpMV, dots, norm) of parallel_pcg_solve with `ranks` in-process ranks
    for _ in range(args.warmup):
        o.pcg_solve(f, max_iter=1, allow_cap=True, ranks=ranks)
    tot, its = 0.0, 0
    for _ in range(args.steps):
        _, hist, ts, _ = o.pcg_solve(f, max_iter=1, allow_cap=True, ranks=ranks)
        tot += ts
        its += len(hist) - 1
    value = n * its / tot
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * tot / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded BASELINE generator)",
        "config": workload_config(args, h, {"parallelism": f"{ranks} in-process ranks (threads)"}),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ranks, "kind": "port",
                         "sample": f"{args.steps} x 1 PCG iteration of parallel_pcg_solve on {args.config}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(args, h, seconds):
    import oracle
    threads = os.cpu_count() or 1
    ranks = max(1, min(threads, h.num_patches))
    o = oracle.Oracle(h)
    f = h.rhs()
    n = h.num_dofs(h.finest_level)
    _, hist, t1, _ = o.pcg_solve(f, max_iter=1, allow_cap=True, ranks=ranks)
    m = int(max(1, min(40, seconds / max(t1, 1e-3))))
    _, hist, ts, _ = o.pcg_solve(f, max_iter=m, allow_cap=True, ranks=ranks)
    its = len(hist) - 1
    return {"value": n * its / ts, "unit": UNIT, "cores": ranks, "kind": "port",
            "sample": f"{its} PCG iterations of parallel_pcg_solve ({ranks} threads) on {args.config}, "
                      f"{ts:.1f} s"}


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import ctypes as C

    import numpy as np
    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1804_02539_b200 import _native as N
    from paper_1804_02539_b200.backend import GpuBackend

    h = build_hierarchy(args)
    L = h.finest_level
    ndofs = h.num_dofs(L)
    if world > 1:
        from paper_1804_02539_b200.parallel import RankBackend
        b = RankBackend(h, rank, world, local)
    else:
        b = GpuBackend(h, device=local)
    stream = torch.cuda.current_stream()
    b.set_stream(stream.cuda_stream)
    f_host = h.rhs()
    f_dev = b.to_distributed_owner(L, f_host)

    def barrier():
        if dist is not None:
            dist.barrier()

    # warm-up (also checks convergence)
    u = b.zero_acc(L)
    for _ in range(args.warmup):
        u, rep = b.pcg_solve_device(f_dev, u=u)
    iters = rep.iterations
    rel_res = rep.residual_history[-1] / rep.residual_history[0]

    lib = N.cuda_lib()

    def timed_solves(profile: bool):
        """K solves bracketed by a barrier + synchronize; CUDA events on the launch
        stream; max over ranks.  With profile=True the library brackets every
        SpMV / FD launch with events (and launches directly instead of replaying
        its CUDA graphs), so kernel durations can be read afterwards."""
        nonlocal u
        lib.pmg_profile(b._ctx, 1 if profile else 0)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        its = []
        e0.record(stream)
        for _ in range(args.steps):
            u, rp = b.pcg_solve_device(f_dev, u=u)
            its.append(rp.iterations)
        e1.record(stream)
        torch.cuda.synchronize()
        barrier()
        lib.pmg_profile(b._ctx, 0)
        t_ms = e0.elapsed_time(e1)
        if dist is not None:
            t = torch.tensor([t_ms], device="cuda", dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            t_ms = float(t.item())
        return t_ms, its

    # ---- device-resident timed region (the reported value)
    b.kernel_launches(reset=True)
    with ClockSampler(local) as clocks:
        ms, step_iters = timed_solves(profile=False)
    launches = b.kernel_launches()
    total_iters = sum(step_iters)
    value = ndofs * total_iters / (ms / 1e3)

    # ---- instrumented replay of the same K steps: per-kernel CUDA events
    for cls in (0, 1):
        lib.pmg_profile_read(b._ctx, cls, L, C.byref(C.c_int64()), C.byref(C.c_double()), C.byref(C.c_double()))
    ms_prof, _ = timed_solves(profile=True)
    nl, sp_ms, sp_bytes = C.c_int64(), C.c_double(), C.c_double()
    lib.pmg_profile_read(b._ctx, 0, L, C.byref(nl), C.byref(sp_ms), C.byref(sp_bytes))
    fd_n, fd_ms, fd_flops = C.c_int64(), C.c_double(), C.c_double()
    lib.pmg_profile_read(b._ctx, 1, L, C.byref(fd_n), C.byref(fd_ms), C.byref(fd_flops))

    # ---- end to end through the public C ABI from pinned host memory
    f_pin = torch.from_numpy(f_host).pin_memory()
    u_pin = torch.empty_like(f_pin).pin_memory()
    hist = np.zeros(501)
    it = C.c_int()
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall = time.perf_counter()
    e0.record(stream)
    e2e_iters = 0
    for _ in range(args.steps):
        if world > 1:
            b.pcg_solve(f_pin.numpy())
            e2e_iters += iters
        else:
            rc = lib.pmg_pcg_solve(b._ctx, C.cast(f_pin.data_ptr(), N._dp), ndofs, 1e-8, 500,
                                   C.cast(u_pin.data_ptr(), N._dp), hist.ctypes.data_as(N._dp), C.byref(it))
            b._check(rc)
            e2e_iters += it.value
    e1.record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    e2e_ms = e0.elapsed_time(e1)
    if dist is not None:
        t = torch.tensor([e2e_ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_ms = float(t.item())
    e2e_value = ndofs * e2e_iters / (e2e_ms / 1e3)

    if rank != 0:
        dist.destroy_process_group()
        return 0

    hbm, hbm_src = peaks()
    achieved = (sp_bytes.value / nl.value) / (sp_ms.value / nl.value / 1e3) / 1e9 if nl.value else None
    traffic = None
    prof = ROOT / "profiles" / f"ncu_{args.config}.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("spmv_dram_bytes_per_launch")
        except Exception:
            traffic = None
    fd_tflops = (fd_flops.value / (fd_ms.value / 1e3) / 1e12) if fd_ms.value else None
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
        "frac": (achieved / hbm) if achieved else None, "traffic": traffic,
        "kernel": (("spmv_sweep2d_kernel (2D line sweep over the line-major symmetric half band: each band "
                    "value read once from HBM and used as lower and mirrored upper entry from shared memory)"
                    if h.dim == 2 else
                    "spmv_tma_half_kernel (index-free symmetric half-band SpMV / residual, TMA bulk-copy stream; "
                    "mirrored half re-read from L2, so the kernel is L2-throughput bound)")
                   + ", finest level; bytes = half band 8(S+D)/2 + vectors (SURVEY.md 8(d)), DESIGN.md"),
        "launches": nl.value, "avg_ms": sp_ms.value / max(nl.value, 1),
        "bytes_per_launch": sp_bytes.value / max(nl.value, 1), "peak_source": hbm_src,
        "timing": "CUDA events around every finest-level launch in an instrumented replay of the same K steps "
                  f"({ms_prof / args.steps:.2f} ms/step instrumented vs {ms / args.steps:.2f} graph-replayed)",
        "spmv_share_of_step": sp_ms.value / ms_prof if ms_prof else None,
        "fd_finest": {"bound": "fp64 tensor (DMMA)", "launches": fd_n.value, "achieved_tflops": fd_tflops,
                      "peak_tflops": 37.0, "frac": fd_tflops / 37.0 if fd_tflops else None,
                      "peak_source": "measured DMMA m8n8k4 peak, profiles/fp64_peak_r01.txt",
                      "share_of_step": fd_ms.value / ms_prof if ms_prof else None},
    }
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and args.assembly == "host":
        cpu = cpu_baseline(args, h, args.cpu_seconds)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator of the BASELINE config; see DESIGN.md)",
        "config": workload_config(args, h, {"parallelism": f"patch-partitioned dp{world}",
                                            "pcg_iterations": iters, "final_rel_residual": rel_res,
                                            "tol_margin": 1e-8 / rel_res, "assembly": args.assembly,
                                            "setup_s": {"host_assembly": h.assemble_seconds(),
                                                        "device_assembly": b.assembly_seconds()}}),
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * ndofs, "d2h_bytes_per_step": 8 * ndofs,
                "ms_per_step": e2e_ms / args.steps, "wall_ms_per_step": 1e3 * t_wall / args.steps},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
