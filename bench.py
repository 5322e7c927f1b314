#!/usr/bin/env python
"""Benchmark of the PCG + V(1,1)-cycle solve path (BASELINE.json metric).

One step = one PCG solve (zero start, V(1,1) preconditioner, tol 1e-8) of the
workload on N GPUs.  Prints ONE JSON line on rank 0.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c5] [--impl reference]

Default workload: BASELINE config 5 (c5), the largest 3D config and the one
the metric's 1-8 GPU figures refer to: 4x4x2 jittered trilinear patches, p=3,
64^3 elements per patch, 9,269,435 dofs, stiffness assembled on the B200.
--gpus N > 1 without a launcher re-executes itself under torchrun (one
process per GPU, NCCL); --config weak runs the weak-scaling boxes
jitter(2,2,1) / (2,2,2) / (4,2,2) / (4,4,2) with 4 patches per GPU.

value     DOF x PCG iterations / s over all ranks (DOF = unique unknowns,
          DofMapper::num_dofs), device-resident load vector; CUDA events on
          the launch stream, max over ranks
e2e       the same metric through the public C ABI (pmg_pcg_solve) from
          pinned host memory: global load vector H2D and global solution D2H
          inside every step
vcycle    CUDA-event time of the graph-replayed V(1,1) cycle (mg_precondition)
          against its roofline time t_roof = sum over the cycle's operations
          of max(bytes / HBM peak, flops / FP64 peak), with
          the band bytes of the symmetric half band the device stores,
          8 B x (S + D) / 2 per level (S = reference CSR entries, D = lattice
          rows)
roofline  the dominant kernel, the finest-level band SpMV: algorithmic bytes
          per launch (half band 8 (S + D) / 2 + 8 B per lattice row for x, y
          and f) / average launch time, timed live with CUDA events around
          every launch in an instrumented replay of the same K steps (kernels
          launched directly, same kernel sequence); shares are taken of the
          graph-replayed step
cpu_baseline  the oracle (CPU restatement of the reference solve path,
          oracle/) with R = min(host threads, patches) in-process ranks on a
          bounded number of PCG iterations of the same workload, on the bands
          the device assembled (downloaded once)
--impl reference  the same oracle on a host-assembled hierarchy (no GPU code
          at all), bounded samples of one PCG iteration, all host threads.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
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
    "weak": "3D weak scaling (BASELINE config 5): 4 jittered trilinear unit-cube patches per GPU, "
            "p=3, 64^3 elements/patch",
}
WEAK_BOXES = {1: (2, 2, 1), 2: (2, 2, 2), 4: (4, 2, 2), 8: (4, 4, 2)}
METRIC = "PCG-MG solve throughput: DOF x PCG iterations per second (one V(1,1) cycle + SpMV per iteration), fp64"
UNIT = "DOF*iter/s"
FP64_PEAK_TFLOPS = 37.0  # measured DMMA m8n8k4 peak, profiles/fp64_peak_r01.txt


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c5")
    ap.add_argument("--levels", type=int, default=None, help="override the refinement depth")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--seed", type=int, default=42)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=15.0, help="target length of the CPU sample")
    ap.add_argument("--operator", default="band", choices=["band", "kronecker"],
                    help="patch operator on the device: the assembled band, or matrix-free as a Kronecker sum "
                         "(axis-aligned affine configs: c1, c3*)")
    ap.add_argument("--assembly", default=None, choices=["host", "device"],
                    help="stiffness assembly of levels >= 1 (default: device for 3D, host for 2D)")
    return ap.parse_args()


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def host_info():
    model = None
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    ram = None
    try:
        for line in Path("/proc/meminfo").read_text().splitlines():
            if line.startswith("MemTotal"):
                ram = round(int(line.split()[1]) / 2**20, 1)
    except OSError:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model, "ram_gb": ram}


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
            time.sleep(0.05)

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


def domain_of(args, world):
    from paper_1804_02539_b200.hierarchy import CONFIGS
    if args.config == "weak":
        if world not in WEAK_BOXES:
            raise SystemExit(f"--config weak: defined for 1, 2, 4, 8 GPUs, not {world}")
        kx, ky, kz = WEAK_BOXES[world]
        return f"jitter({kx},{ky},{kz})", 3, 2, 5
    return CONFIGS[args.config]


def build_hierarchy(args, world=1, threads=None, assembly=None, rhs="default"):
    from paper_1804_02539_b200.hierarchy import Hierarchy
    dom, p, n0, lv = domain_of(args, world)
    if args.levels is not None:
        lv = args.levels
    return Hierarchy(dom, p, lv, n0=n0, seed=args.seed, threads=threads, assembly=assembly or "host",
                     operator=args.operator, rhs=rhs)


def default_assembly(args):
    if args.assembly:
        return args.assembly
    return "device" if args.config in ("c4", "c5", "weak") else "host"


def workload_config(args, h, world, extra=None):
    L = h.finest_level
    cfg = {
        "workload": f"{args.config}: {WORKLOADS.get(args.config, args.config)}; PCG + V(1,1), tol 1e-8, zero start",
        "domain": h.domain, "dofs": h.num_dofs(L), "levels": h.num_levels, "degree": h.degree,
        "patches": h.num_patches, "elements_per_patch_dir": h.elements(L), "coarsest_elements": h.elements(0),
        "stored_band_entries_finest": h.stored_entries(L),
        "l2": "inputs larger than L2 (finest band alone exceeds 126 MB); no flush"
        if h.stored_entries(L) * 4 > 126e6 else "inputs smaller than L2; no flush (solve is latency bound)",
        "parallelism": f"patch-partitioned dp{world} (contiguous_partition, parallel.cpp:181-198)",
    }
    if extra:
        cfg.update(extra)
    return cfg


# ------------------------------------------------------------------ roofline of one V-cycle
def vcycle_roofline(h, hbm_gbs, fp64_tflops):
    """Roofline time of one V(1,1) cycle: per level l >= 1 two residual
    SpMVs (8 B (S + D)/2 half band + 24 B D vectors), two fast-diagonalization
    applications (16 B per interior/face dof; 4 prod(m) sum(m) flops per
    piece), restriction (8 D_l + 8 D_{l-1}), prolongation (8 D_{l-1} + 16 D_l),
    two axpys (24 B D_l); level 0 the coarse GEMV (8 N0^2).  The FD term takes
    the max of its bytes and flops; everything else is HBM-bound."""
    bw = hbm_gbs * 1e9
    pk = fp64_tflops * 1e12
    t = 0.0
    bytes_total, flops_total = 0.0, 0.0
    for lvl in range(1, h.num_levels):
        D = h.lattice_size(lvl) * h.num_patches
        Dc = h.lattice_size(lvl - 1) * h.num_patches
        S = h.stored_entries(lvl)
        spmv = 8.0 * (S + D) / 2 + 24.0 * D
        fd_dofs, fd_flops = 0.0, 0.0
        for pc in h.pieces(lvl):
            if pc.kind in (0, 1):  # interior and face pieces: fast diagonalization
                dims = [pc.dims[a] for a in range(pc.naxes)]
                prod = 1.0
                for m in dims:
                    prod *= m
                fd_dofs += prod
                fd_flops += 4.0 * prod * sum(dims)
        other = (8.0 * D + 8.0 * Dc) + (8.0 * Dc + 16.0 * D) + 2 * 24.0 * D
        t += 2 * spmv / bw + 2 * max(16.0 * fd_dofs / bw, fd_flops / pk) + other / bw
        bytes_total += 2 * spmv + 2 * 16.0 * fd_dofs + other
        flops_total += 2 * fd_flops
    n0 = h.num_dofs(0)
    t += 8.0 * n0 * n0 / bw
    bytes_total += 8.0 * n0 * n0
    return t, bytes_total, flops_total


# ------------------------------------------------------------------ reference arm
def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    threads = os.cpu_count() or 1
    t0 = time.perf_counter()
    h = build_hierarchy(args, world=args.gpus, threads=threads, assembly="host")
    t_setup = time.perf_counter() - t0
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
        "scaling": "weak" if args.config == "weak" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded BASELINE generator)",
        "config": workload_config(args, h, args.gpus, {"cpu_parallelism": f"{ranks} in-process ranks (threads)",
                                                       "assembly": "host", "host_setup_s": t_setup,
                                                       "host": host_info()}),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": ranks, "kind": "port",
                         "sample": f"{args.steps} x 1 PCG iteration of parallel_pcg_solve on {args.config}"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(args, h, b, seconds, f=None):
    import oracle
    threads = os.cpu_count() or 1
    ranks = max(1, min(threads, h.num_patches))
    t_dl = h.adopt_device_bands(b) if h.assembly == "device" else 0.0
    o = oracle.Oracle(h)
    if f is None:
        f = h.rhs()
    n = h.num_dofs(h.finest_level)
    _, hist, t1, _ = o.pcg_solve(f, max_iter=1, allow_cap=True, ranks=ranks)
    m = int(max(1, min(40, seconds / max(t1, 1e-3))))
    _, hist, ts, _ = o.pcg_solve(f, max_iter=m, allow_cap=True, ranks=ranks)
    its = len(hist) - 1
    src = ("on the bands the device assembled (downloaded once, %.1f s)" % t_dl) if t_dl else "on host-assembled bands"
    return {"value": n * its / ts, "unit": UNIT, "cores": ranks, "kind": "port",
            "sample": f"{its} PCG iterations of parallel_pcg_solve ({ranks} threads) on {args.config}, "
                      f"{ts:.1f} s, {src}",
            "host": host_info(), "residual_history_head": [float(x) for x in hist[:4]]}


def free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(args):
    """--gpus N > 1 without a launcher: re-execute under torchrun, one process
    per GPU (NCCL), NCCL_DEBUG=INFO to stderr."""
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr=127.0.0.1", f"--master-port={free_port()}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.call(cmd, env=env)


# ------------------------------------------------------------------ our arm
def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return relaunch(args)
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
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_1804_02539_b200 import _native as N
    from paper_1804_02539_b200.backend import GpuBackend

    assembly = default_assembly(args)
    threads = max(1, (os.cpu_count() or 1) // world)
    t0 = time.perf_counter()
    # with device assembly the load vector is assembled on the device as well
    # (pmg_assemble_load): the host quadrature loop is 13 s at c4, 50 s at c5
    device_load = assembly == "device"
    h = build_hierarchy(args, world=world, threads=threads, assembly=assembly,
                        rhs="zero" if device_load else "default")
    t_setup = time.perf_counter() - t0
    L = h.finest_level
    ndofs = h.num_dofs(L)
    if world > 1:
        from paper_1804_02539_b200.parallel import RankBackend
        b = RankBackend(h, rank, world, local)
    else:
        b = GpuBackend(h, device=local)
    # a dedicated stream: every launch of the library and every timing event
    # go to it (the legacy default stream would not order against the
    # library's non-blocking streams)
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    b.set_stream(stream.cuda_stream)
    if device_load:
        f_dev = b.assemble_load("default")
        f_host = b.gather_global(L, f_dev)  # replica sums of this rank's patches
        if dist is not None:  # the global load vector: the sum over the ranks' shares
            t = torch.from_numpy(f_host).cuda()
            dist.all_reduce(t)
            f_host = t.cpu().numpy()
    else:
        f_host = h.rhs()
        f_dev = b.to_distributed_owner(L, f_host)

    def barrier():
        if dist is not None:
            dist.barrier()

    def max_over_ranks(ms):
        if dist is None:
            return ms
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    # warm-up (captures the solve graph, checks convergence)
    u = b.zero_acc(L)
    for _ in range(args.warmup):
        u, rep = b.pcg_solve_device(f_dev, u=u)
    iters = rep.iterations
    rel_res = rep.residual_history[-1] / rep.residual_history[0]

    lib = N.cuda_lib()

    def timed_solves(profile: bool):
        """K solves bracketed by a barrier + synchronize; CUDA events on the launch
        stream; max over ranks.  With profile=True the library brackets every
        timed kernel class with events and launches directly (same kernels)."""
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
        return max_over_ranks(e0.elapsed_time(e1)), its

    # ---- device-resident timed region (the reported value)
    b.kernel_launches(reset=True)
    with ClockSampler(local) as clocks:
        ms, step_iters = timed_solves(profile=False)
    launches = b.kernel_launches()
    total_iters = sum(step_iters)
    value = ndofs * total_iters / (ms / 1e3)
    ms_step = ms / args.steps

    # ---- V-cycle: CUDA events around graph-replayed mg_precondition calls
    r_dev = b.to_distributed_owner(L, f_host)
    z_dev = b.zero_acc(L)
    for _ in range(2):
        b.precondition(r_dev, out=z_dev)
    nv = max(5, 2 * args.steps)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for _ in range(nv):
        b.precondition(r_dev, out=z_dev)
    e1.record(stream)
    torch.cuda.synchronize()
    v_ms = max_over_ranks(e0.elapsed_time(e1)) / nv
    hbm, hbm_src = peaks()
    # roofline of this rank's share: the V-cycle of the whole problem / world
    t_roof, v_bytes, v_flops = vcycle_roofline(h, hbm, FP64_PEAK_TFLOPS)
    t_roof_ms = 1e3 * t_roof / world

    # ---- instrumented replay of the same K steps: per-class CUDA events
    levels = range(h.num_levels)
    for cls in range(6):
        for lv in levels:
            lib.pmg_profile_read(b._ctx, cls, lv, C.byref(C.c_int64()), C.byref(C.c_double()), C.byref(C.c_double()))
    ms_prof, _ = timed_solves(profile=True)
    cls_ms = {}
    per = {}
    for cls in range(6):
        tot = 0.0
        for lv in levels:
            nl, t, w = C.c_int64(), C.c_double(), C.c_double()
            lib.pmg_profile_read(b._ctx, cls, lv, C.byref(nl), C.byref(t), C.byref(w))
            tot += t.value
            per[(cls, lv)] = (nl.value, t.value, w.value)
        cls_ms[cls] = tot
    sp_n, sp_ms, sp_bytes = per[(0, L)]
    fd_n, fd_ms, fd_flops = per[(1, L)]

    # ---- end to end through the public C ABI from pinned host memory
    f_pin = torch.from_numpy(f_host).pin_memory()
    u_pin = torch.empty_like(f_pin).pin_memory()
    hist = np.zeros(501)
    it = C.c_int()

    def e2e_solve():
        if world > 1:
            _, rp = b.pcg_solve(f_pin.numpy())
            return rp.iterations
        rc = lib.pmg_pcg_solve(b._ctx, C.cast(f_pin.data_ptr(), N._dp), ndofs, 1e-8, 500,
                               C.cast(u_pin.data_ptr(), N._dp), hist.ctypes.data_as(N._dp), C.byref(it))
        b._check(rc)
        return it.value

    e2e_solve()  # captures the host-vector solve graph
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_wall = time.perf_counter()
    e0.record(stream)
    e2e_iters = 0
    for _ in range(args.steps):
        e2e_iters += e2e_solve()
    e1.record(stream)
    torch.cuda.synchronize()
    t_wall = time.perf_counter() - t_wall
    e2e_ms = max_over_ranks(e0.elapsed_time(e1))
    e2e_value = ndofs * e2e_iters / (e2e_ms / 1e3)

    if rank != 0:
        dist.destroy_process_group()
        return 0

    achieved = (sp_bytes / sp_n) / (sp_ms / sp_n / 1e3) / 1e9 if sp_n else None
    traffic, traffic_src = None, None
    prof = ROOT / "profiles" / f"ncu_{args.config}.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get("spmv_dram_bytes_per_launch")
            traffic_src = str(prof.relative_to(ROOT)) + " (ncu --set full of the same kernel on this config)"
        except Exception:
            traffic = None
    fd_tflops = (fd_flops / (fd_ms / 1e3) / 1e12) if fd_ms else None
    steps = args.steps
    # kernel time per graph-replayed step: the instrumented replay runs the
    # same kernel sequence, so its per-step kernel time is comparable
    names = {0: "band_spmv", 1: "fd_passes", 2: "transfers", 3: "interface_pieces_side_stream", 4: "dots_accumulate",
             5: "coarse_solve"}
    breakdown = {names[c]: {"ms_per_step": cls_ms[c] / steps, "share_of_step": cls_ms[c] / steps / ms_step}
                 for c in range(6)}
    if args.operator == "kronecker":
        kernel_desc = ("kron2d_kernel / kron3d_axis*_kernel (matrix-free Kronecker-sum operator, PMG_BAND_KRONECKER), "
                       "finest level; bytes = 8 B per lattice row for x, y (and f) + 4 B for the Dirichlet map")
    else:
        kernel_desc = (("spmv_sweep2d_kernel (2D line sweep over the line-major symmetric half band: each band "
                        "value read once from HBM and used as lower and mirrored upper entry from shared memory)"
                        if h.dim == 2 else
                        "spmv_sweep3d_kernel (3D plane sweep over the plane-major symmetric half band: each band "
                        "value read once from HBM and used as lower and mirrored upper entry from shared memory)")
                       + ", finest level; bytes = half band 8 (S + D) / 2 + 8 B per lattice row for x, y (and f), "
                         "SURVEY.md 8(d), DESIGN.md 3")
    # per level: launches and ms per step of every timed class, and the SpMV's
    # fraction of the HBM peak on its algorithmic bytes
    per_level = {}
    for lv in levels:
        row = {}
        for c in range(6):
            nl_, t_, w_ = per[(c, lv)]
            if nl_:
                row[names[c]] = {"launches_per_step": nl_ / steps, "ms_per_step": t_ / steps}
                if c == 0 and t_ > 0:
                    row[names[c]]["hbm_frac"] = (w_ / (t_ / 1e3) / 1e9) / hbm
                if c == 1 and t_ > 0:
                    row[names[c]]["tflops"] = w_ / (t_ / 1e3) / 1e12
        per_level[str(lv)] = row
    roofline = {
        "bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s",
        "frac": (achieved / hbm) if achieved else None, "traffic": traffic, "traffic_source": traffic_src,
        "kernel": kernel_desc,
        "launches": sp_n, "avg_ms": sp_ms / max(sp_n, 1), "bytes_per_launch": sp_bytes / max(sp_n, 1),
        "peak_source": hbm_src,
        "timing": "CUDA events around every finest-level launch in an instrumented replay of the same K steps "
                  f"({ms_prof / steps:.2f} ms/step instrumented vs {ms_step:.2f} graph-replayed)",
        "share_of_step": sp_ms / steps / ms_step,
        "fd_finest": {"bound": "fp64 tensor (DMMA)", "launches": fd_n, "achieved_tflops": fd_tflops,
                      "peak_tflops": FP64_PEAK_TFLOPS, "frac": fd_tflops / FP64_PEAK_TFLOPS if fd_tflops else None,
                      "peak_source": "measured DMMA m8n8k4 peak on a B200, profiles/fp64_peak_r01.txt",
                      "share_of_step": fd_ms / steps / ms_step},
        "breakdown": breakdown,
        "per_level": per_level,
    }
    vcycle = {
        "ms": v_ms, "t_roof_ms": t_roof_ms, "frac": t_roof_ms / v_ms,
        "dofs_per_s": ndofs / (v_ms / 1e3),
        "roofline_dofs_per_s": ndofs / (t_roof_ms / 1e3),
        "bytes": v_bytes, "fd_flops": v_flops,
        "share_of_step": v_ms * total_iters / steps / ms_step,
        "timing": f"CUDA events around {nv} graph-replayed mg_precondition calls (pmg_precondition), max over ranks",
        "model": "t_roof = sum of max(bytes / HBM peak, flops / FP64 peak) per operation; half-band SpMV bytes "
                 "8 (S + D) / 2 + 24 D per residual, SURVEY.md 8(d); divided by the GPU count",
    }
    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args, h, b, args.cpu_seconds, f_host)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "weak" if args.config == "weak" else "strong", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded generator of the BASELINE config; see DESIGN.md)",
        "config": workload_config(args, h, world, {
            "pcg_iterations": iters, "final_rel_residual": rel_res, "tol_margin": 1e-8 / rel_res,
            "assembly": assembly, "operator": args.operator,
            "setup_s": {"host_setup": t_setup, "host_assembly": h.assemble_seconds(),
                        "device_assembly": b.assembly_seconds(), "device_load_vector": b.load_seconds()},
            "solve_ms": ms_step}),
        "vcycle": vcycle,
        "roofline": roofline,
        "cpu_baseline": cpu,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": 8 * ndofs, "d2h_bytes_per_step": 8 * ndofs,
                "ms_per_step": e2e_ms / steps, "wall_ms_per_step": 1e3 * t_wall / steps},
        "clocks": clocks.summary(),
        "gpu_launches": launches,
    }
    print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
