"""Benchmark of the B200 Hermite time step (driver contract: one JSON line on rank 0).

Workload (BASELINE.json configs[2], the headline metric): 3D periodic advection,
Hermite order m = N = 3, 512^3 cells per GPU, plane-wave initial data (device
init, synthetic), cfl 0.9, q = 21, fused monolithic kernel, FP64.  A "step" is one
full time step = two half steps (primary -> dual -> primary).

    value  = DOF-updates/s = M^3 (N+1)^3 * steps * n_ranks / max-over-ranks device time
    e2e    = same metric through the package API with the state in pinned HOST
             memory: every step uploads the field, steps it, and reads it back
    roofline = dominant kernel (sep_fused) algorithmic bytes 16 (N+1)^3 per node per
             launch / mean CUDA-event launch time, against MEASURED_PEAKS.json hbm_gbs
    cpu_baseline = the CPU oracle port (oracle/h3_oracle.c, OpenMP, all host cores)
             on a bounded sample of the same per-cell work

`--impl reference` times the reference's CPU algorithm (the oracle port, since the
Python reference cannot travel to the GPU box) on rank 0 and prints its line.
Multi-GPU (torchrun): slab decomposition along x3, 512^3 per rank (weak scaling),
one-plane NCCL halo exchange per half step overlapped with interior cells.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "DOF-updates/sec per time step (FP64) at m=3, 512^3; % HBM roofline; 1/2/4/8 GPU"
UNIT = "DOF-updates/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--order", type=int, default=3)
    ap.add_argument("--cells", type=int, default=512, help="cells per axis (per GPU along x3)")
    ap.add_argument("--mode", default="fused", choices=["fused", "two_pass"])
    ap.add_argument("--variant", default="separable", choices=["separable", "literal", "auto"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-extras", action="store_true",
                    help="skip the secondary configs (two-kernel 512^3 / 128^3, m=5 256^3)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--strong", type=int, default=0, metavar="M",
                    help="strong scaling: one M^3 grid split over the N ranks (configs[4]: M = 1024 on 8 GPUs); "
                         "default: weak scaling with --cells^3 per GPU")
    ap.add_argument("--halo", default="auto", choices=["auto", "nccl", "p2p"],
                    help="N>1 halo: in-kernel reads of the neighbour plane over NVLink (p2p), NCCL copy, "
                         "or auto (p2p verified against NCCL at start-up, else NCCL)")
    ap.add_argument("--backend", default="nccl", choices=["nccl", "gloo"],
                    help="process-group backend for N>1 (gloo: test the multi-rank path on one GPU)")
    return ap.parse_args()


# ----------------------------------------------------------------------------- helpers

def measured_traffic(order_n, cells, mode, variant):
    """DRAM bytes per launch of the dominant kernel from the committed ncu capture
    (profiles/*_summary.json), when that capture is of this exact workload."""
    if (order_n, cells, mode, variant) != (3, 512, "fused", "separable"):
        return None, None
    p = ROOT / "profiles" / "r02_fused3_512_sep_fused_summary.json"
    if not p.exists():
        return None, None
    d = json.loads(p.read_text())
    gb = float(d["dram__bytes_read.sum"]["value"]) + float(d["dram__bytes_write.sum"]["value"])
    return gb * 1e9, str(p.relative_to(ROOT))


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled while the timed region runs."""

    FIELDS = ["clocks.sm", "clocks.max.sm", "clocks_event_reasons.hw_slowdown",
              "clocks_event_reasons.hw_thermal_slowdown", "clocks_event_reasons.sw_thermal_slowdown",
              "clocks_event_reasons.sw_power_cap"]

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), "--query-gpu=" + ",".join(self.FIELDS),
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) != len(self.FIELDS):
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(names, parts[2:]):
                if val.lower().startswith("active"):
                    reasons.add(name)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_oracle_rate(order_n, cells, seconds_budget):
    """DOF-updates/s of the oracle port (bit-exact C restatement of the reference's
    numba kernels) on a bounded sample: full steps of a periodic plane-wave grid."""
    from oracle import refmodel as rm
    rm.build()
    import numpy as np
    n3 = (order_n + 1) ** 3
    state = rm.init_field(rm.plane_wave_terms(), cells, (1.0, 1.0, 1.0), order_n)
    scratch = np.zeros_like(state)
    dt = rm.select_dt(cells)
    t0 = time.perf_counter()
    rm.full_step(state, scratch, order_n, cells, (1.0, 1.0, 1.0), dt)
    one = time.perf_counter() - t0
    steps = max(1, min(50, int(seconds_budget / max(one, 1e-6))))
    t0 = time.perf_counter()
    for _ in range(steps):
        rm.full_step(state, scratch, order_n, cells, (1.0, 1.0, 1.0), dt)
    wall = time.perf_counter() - t0
    dofs = cells[0] * cells[1] * cells[2] * n3
    return dofs * steps / wall, {
        "cores": rm.max_threads(), "steps": steps, "wall_s": wall,
        "sample": f"{steps} full step(s) of m={order_n} {cells[0]}x{cells[1]}x{cells[2]} periodic "
                  f"plane wave, fused (the per-cell work of the {METRIC.split(';')[0]} workload; "
                  f"CPU throughput is grid-size independent), {wall:.1f} s"}


def cpu_model():
    """Host CPU model name (the reference's perf report names it: SURVEY 8(d))."""
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def cpu_sample_cells(order_n):
    return {0: (128,) * 3, 1: (64,) * 3, 2: (48,) * 3, 3: (48,) * 3, 4: (32,) * 3, 5: (24,) * 3}[order_n]


# ----------------------------------------------------------------------------- reference arm

def run_reference(args, rank, world):
    if rank != 0:
        return
    # torchrun exports OMP_NUM_THREADS=1 per rank; the reference arm uses every host core it
    # can (set before the oracle's OpenMP runtime starts: torch is not imported on this arm)
    os.environ["OMP_NUM_THREADS"] = str(len(os.sched_getaffinity(0)))
    order_n = args.order
    cells = cpu_sample_cells(order_n)
    rates = []
    info = None
    for _ in range(max(1, args.warmup if args.warmup < 2 else 1)):
        cpu_oracle_rate(order_n, (8, 8, 8), 0.1)
    budget = max(2.0, min(args.cpu_seconds, 120.0 / max(1, args.steps)))
    for _ in range(max(1, args.steps)):
        r, info = cpu_oracle_rate(order_n, cells, budget)
        rates.append(r)
    value = statistics.median(rates)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (plane wave)",
        "config": {"workload": f"m={order_n} {args.cells}^3 periodic advection, reference CPU algorithm",
                   "order_m": order_n, "cells": args.cells, "sampled_cells": list(cells)},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": info["cores"], "kind": "port", "cpu": cpu_model(),
                         "sample": info["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- our arm

def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_1609_09841_b200 as hb
    from paper_1609_09841_b200 import _native, distributed as hd

    torch.cuda.set_device(local % torch.cuda.device_count())
    if world > 1:
        if args.backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group("gloo")
    order_n, m = args.order, args.cells
    n3 = (order_n + 1) ** 3
    peak_gbs, peak_src = peaks()

    if world > 1:
        gcells = (args.strong,) * 3 if args.strong else (m, m, m * world)
        solver = hd.SlabSolver(gcells, order_n, hb.StepConfig(mode=args.mode, variant=args.variant),
                               lengths=(1.0, 1.0, 1.0) if args.strong else (1.0, 1.0, float(world)), halo=args.halo)
        solver.init(hb.plane_wave())
        step_fn = solver.step
        launches_per_step = solver.launches_per_step
        kernel_events = solver.kernel_events
    else:
        grid = hb.GridSpec((m, m, m))
        cfg = hb.StepConfig(mode=args.mode, variant=args.variant)
        ops = hb.OperatorSet.for_grid(grid, order_n)
        state = hb.init_field(hb.plane_wave(), grid, order_n)
        scratch = hb.DofField.empty(grid.with_parity("dual"), order_n)
        dt = hb.select_dt(grid, cfg)
        kernel_times = []
        stream = torch.cuda.current_stream()

        def step_fn(timed=False):
            for src, dst in ((state, scratch), (scratch, state)):
                if timed:
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(stream)
                hb.half_step(src, dst, cfg, ops, dt=dt, _flag=flags[0:1], _check=False)
                if timed:
                    e1.record(stream)
                    kernel_times.append((e0, e1))

        flags = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        launches_per_step = 2 if args.mode == "fused" else 4 * math.ceil(m / hb.pipeline._coeff_chunk_planes(
            grid, order_n, 8, None))
        kernel_events = kernel_times

    for _ in range(args.warmup):
        step_fn()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    with ClockSampler(local % torch.cuda.device_count()) as clocks:
        kernel_events.clear()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = torch.cuda.Event(enable_timing=True)
        t1 = torch.cuda.Event(enable_timing=True)
        t0.record()
        for _ in range(args.steps):
            step_fn(timed=True)
        t1.record()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ms = t0.elapsed_time(t1)
    ms_t = torch.tensor([ms], dtype=torch.float64, device="cuda" if args.backend == "nccl" else "cpu")
    if world > 1:
        dist.all_reduce(ms_t, op=dist.ReduceOp.MAX)
    ms_max = float(ms_t.item())
    dofs_per_step = (args.strong ** 3 if args.strong and world > 1 else m * m * m * world) * n3
    value = dofs_per_step * args.steps / (ms_max / 1e3)

    # dominant-kernel roofline: mean launch time of the half-step kernel
    launch_ms = statistics.mean(a.elapsed_time(b) for a, b in kernel_events) if kernel_events else None
    cells_local = dofs_per_step // world // n3
    if world > 1 and solver.halo != "p2p":  # the timed launch is the interior: L-1 of the L cell planes
        cells_local = cells_local * (solver.local - 1) // solver.local
    alg_bytes = 16 * n3 * cells_local if args.mode == "fused" else 16 * (n3 + (2 * order_n + 2) ** 3) * cells_local
    achieved = alg_bytes / (launch_ms / 1e3) / 1e9 if launch_ms else None

    if world == 1:
        finite = int(flags[0].item()) == -1
    else:
        try:
            solver.check()  # collective: every rank sees the same verdict
            finite = True
        except hb.InstabilityError:
            finite = False
    traffic, traffic_src = measured_traffic(order_n, m, args.mode, args.variant)
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_max / args.steps, "higher_is_better": True,
        "scaling": "strong" if args.strong and world > 1 else "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic: plane-wave initial data generated on device (h3_init_separable)",
        "config": {"workload": f"m={order_n}, {m}^3 cells per GPU, {args.mode} "
                               f"{'monolithic' if args.mode == 'fused' else 'two-kernel'} "
                               f"({args.variant}) half-step kernels, periodic advection, cfl 0.9, q={3 * (2 * order_n + 1)}",
                   "order_m": order_n,
                   "cells_per_gpu": [args.strong, args.strong, args.strong // world] if args.strong and world > 1 else [m, m, m],
                   "global_cells": [args.strong] * 3 if args.strong and world > 1 else [m, m, m * world],
                   "mode": args.mode, "variant": args.variant, "parallelism": f"slab-x3 x{world}",
                   "halo": (solver.halo + (f" ({solver.halo_note})" if solver.halo_note else "")) if world > 1 else None,
                   "l2": f"inputs larger than L2 ({dofs_per_step // world * 8 / 1e9:.1f} GB per field vs 126 MB L2)"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                     "frac": (achieved / peak_gbs) if achieved else None, "traffic": traffic,
                     "traffic_unit": "DRAM bytes per launch (ncu dram__bytes_read+write)",
                     "traffic_source": traffic_src,
                     "kernel": ("sep_fused_dmma3_kernel (DMMA m8n8k4, 8x7 tile, 16 warps, TMA row loads, x3/x1 plane pipelining, "
                                 "column-band tile rasterisation)" if order_n == 3
                                else ("sep_fused_dmma_ws_kernel (DMMA cell-pair, warp-specialised)" if order_n == 5
                                      else f"sep_fused_kernel<{order_n}>")) if args.mode == "fused" else "recon+evolve",
                     "algorithmic_bytes_per_launch": alg_bytes, "mean_launch_ms": launch_ms,
                     "peak_source": peak_src},
        "gpu_launches": launches_per_step * args.steps,
        # also the per-half-step node rate (nodes updated per second, whole job)
        "node_updates_per_s_per_half_step": (dofs_per_step // n3) / (ms_max / args.steps / 2 / 1e3),
        "finite": finite,
    }
    result["clocks"] = clocks.summary()

    # ---- e2e through the package API with host-resident state ------------------------------
    print(f"[bench] value {value:.4e} DOF-updates/s, kernel {launch_ms} ms", file=sys.stderr, flush=True)
    if not args.no_e2e:
        local_bytes = dofs_per_step // world * 8
        room = host_room(local_bytes)
        if world > 1:  # every rank must take part (the streamed step exchanges halo planes)
            ok = torch.tensor([1 if room is None else 0], dtype=torch.int64,
                              device="cuda" if args.backend == "nccl" else "cpu")
            dist.all_reduce(ok, op=dist.ReduceOp.MIN)
            if room is None and int(ok.item()) == 0:
                room = "another rank lacks host memory for its slab"
        if room is not None:
            result["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                             "error": room}
        else:
            if world == 1:
                del scratch
                scratch = None
                e2e_args = (state, grid, cfg, dt, None)
            else:
                e2e_args = (solver.state, solver.grid, solver.cfg, solver.dt, solver)
            torch.cuda.empty_cache()
            try:
                fstate, fgrid, fcfg, fdt, fsolver = e2e_args
                del e2e_args
                result["e2e"] = e2e_host(hb, torch, fstate, fgrid, order_n, fcfg, fdt, args.e2e_steps, dofs_per_step,
                                         solver=fsolver, dist=dist)
                del fstate
            except (RuntimeError, MemoryError, ValueError) as exc:  # e.g. pinning failed, two-pass mode
                result["e2e"] = {"value": None, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                                 "error": f"{type(exc).__name__}: {exc}"[:300]}
        print(f"[bench] e2e {result['e2e']}", file=sys.stderr, flush=True)
    # ---- CPU baseline (rank 0, N = 1) ----------------------------------------------------------
    if world == 1 and not args.no_cpu:
        try:
            rate, info = cpu_oracle_rate(order_n, cpu_sample_cells(order_n), args.cpu_seconds)
            result["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": info["cores"], "kind": "port",
                                      "cpu": cpu_model(), "sample": info["sample"]}
        except (OSError, RuntimeError, subprocess.CalledProcessError) as exc:
            result["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": 0, "kind": "port",
                                      "error": f"{type(exc).__name__}: {exc}"[:300]}
    if world == 1 and not args.no_extras:
        del state, scratch
        torch.cuda.empty_cache()
        result["extras"] = extras(hb, torch, order_n, peak_gbs)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        dist.destroy_process_group()


def host_room(local_bytes):
    """None when this node's free host memory holds every local rank's pinned field copy
    (with 25 % headroom), else the reason: pinning more than is free would invite the OOM
    killer and lose the whole bench line."""
    try:
        with open("/proc/meminfo") as fh:
            info = {l.split(":")[0]: int(l.split()[1]) * 1024 for l in fh if ":" in l}
        free = info.get("MemAvailable", 0)
    except (OSError, ValueError):
        return "cannot read /proc/meminfo"
    ranks_here = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    need = int(1.25 * local_bytes * ranks_here)
    return None if need <= free else f"host memory: {need / 1e9:.0f} GB needed, {free / 1e9:.0f} GB available"


def e2e_host(hb, torch, state, grid, order_n, cfg, dt, steps, dofs_per_step, solver=None, dist=None):
    """Host-resident state through the package API (HostStepper, the drop-in for the
    reference's full_step on a host field): every step uploads the whole primary field (N > 1:
    each rank its x3 slab) from pinned host memory, steps it and writes it back, with the
    transfers and kernels of successive x3 chunks overlapped and (N > 1) the slab halo planes
    exchanged over NCCL; the step's result (instability flags) is read back.  Wall time, max
    over ranks."""
    dof_field = state if solver is None else None
    src = state.tensor if solver is None else state
    try:
        host = torch.empty(src.shape, dtype=torch.float64, pin_memory=True)
        pinned = True
    except RuntimeError:
        host = torch.empty(src.shape, dtype=torch.float64)
        pinned = False
    host.copy_(src)
    del src, state  # (a slab view keeps the solver's field alive until the caller drops it: HBM has room)
    if solver is None:
        dof_field.tensor = None  # free HBM: the streamed step keeps only a few chunks on the device
    else:
        solver.close()
        solver.bufs = None
    torch.cuda.empty_cache()
    world = dist.get_world_size() if solver is not None else 1
    stepper = hb.HostStepper(host, grid, order_n, cfg)
    stepper.step(dt=dt)  # warm-up (allocations, first launches)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for k in range(steps):
        stepper.step(dt=dt, step_index=k)  # ends with the D2H read of the step's flags
    wall = time.perf_counter() - t0
    if world > 1:
        w = torch.tensor([wall], dtype=torch.float64,
                         device="cuda" if dist.get_backend() == "nccl" else "cpu")
        dist.all_reduce(w, op=dist.ReduceOp.MAX)
        wall = float(w.item())
    return {"value": dofs_per_step * steps / wall, "unit": UNIT, "h2d_bytes_per_step": stepper.h2d_bytes * world,
            "d2h_bytes_per_step": (stepper.d2h_bytes + 16 * len(stepper.chunks)) * world, "steps": steps,
            "pinned": pinned, "chunks": len(stepper.chunks), "wall_s": wall,
            "api": "paper_1609_09841_b200.HostStepper.step on a host-resident field (chunked H2D -> fused "
                   "half steps -> D2H, overlapped on three streams"
                   + (f"; {world} ranks, each streaming its x3 slab, halo planes over "
                      f"{dist.get_backend()})" if world > 1 else ")")}


def extras(hb, torch, order_n, peak_gbs):
    """Secondary measurements (device-resident state, CUDA events), each against its own
    algorithmic-byte roofline: fused 16 (N+1)^3 B and two-kernel 16 ((N+1)^3 + (2N+2)^3) B per
    node per half step.  Covers the north-star targets (m=3 512^3 fused AND two-kernel) and
    BASELINE configs[1] (m=3 128^3 two-kernel) and configs[3] (m=5 256^3 both forms)."""
    out = {}
    for (n, m, mode, k) in ((3, 512, "two_pass", 2), (3, 128, "two_pass", 10), (3, 128, "fused", 10),
                            (5, 256, "fused", 5), (5, 256, "two_pass", 3)):
        try:
            out[f"m{n}_{m}^3_{mode}"] = _extra(hb, torch, n, m, mode, k, peak_gbs)
        except (RuntimeError, MemoryError) as exc:  # a secondary line must never cost the main one
            out[f"m{n}_{m}^3_{mode}"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        torch.cuda.empty_cache()
    return out


def _extra(hb, torch, n, m, mode, k, peak_gbs):
    """One secondary configuration: device-resident field, CUDA events, its own roofline."""
    grid = hb.GridSpec((m, m, m))
    cfg = hb.StepConfig(mode=mode, variant="separable")
    ops = hb.OperatorSet.for_grid(grid, n)
    st = hb.init_field(hb.plane_wave(), grid, n)
    sc = hb.DofField.empty(grid.with_parity("dual"), n)
    hb.run_steps(st, sc, cfg, ops, 1)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    hb.run_steps(st, sc, cfg, ops, k)
    b.record()
    torch.cuda.synchronize()
    ms = a.elapsed_time(b) / k
    rate = m ** 3 * (n + 1) ** 3 / (ms / 1e3)
    per_dof = 32 if mode == "fused" else 32 * (1 + 8)  # bytes per DOF-update (two half steps)
    gbs = rate * per_dof / 1e9
    print(f"[bench] extra m{n} {m}^3 {mode}: {rate:.3e} DOF-updates/s, {gbs:.0f} GB/s "
          f"({100 * gbs / peak_gbs:.1f}% of HBM)", file=sys.stderr, flush=True)
    del st, sc
    return {"dof_updates_per_s": rate, "ms_per_step": ms, "alg_GBps": gbs, "hbm_frac": gbs / peak_gbs,
            "steps": k}


if __name__ == "__main__":
    main()
